"""nu_sigma by its plain definition (Eq. 1.1).

nu_sigma(A, B) = #{i : lambda_i < sigma} for A x = lambda B x with A
symmetric and B symmetric positive definite.  The eigenvalues come from a
library routine (scipy.linalg.eigh -> LAPACK dsygvd), used as a step.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


def eigvals_pencil(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """All eigenvalues of the dense pencil (A, B), ascending."""
    return sla.eigh(A, B, eigvals_only=True)


def nu_eig(A: np.ndarray, B: np.ndarray, sigma, eigvals=None):
    """Count of eigenvalues strictly below sigma (scalar or array of shifts)."""
    w = eigvals_pencil(A, B) if eigvals is None else np.asarray(eigvals)
    s = np.asarray(sigma, dtype=np.float64)
    return np.searchsorted(w, s, side="left") if s.ndim else int(np.searchsorted(w, s, side="left"))
