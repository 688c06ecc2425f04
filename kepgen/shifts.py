"""Shift placement for tests and benchmarks (input generation only).

SURVEY.md §8(c) reading 11: sigma_i = lo + (i + 1/2)(hi - lo)/m over the
spectrum interval.  ``spectral_bounds`` gives [lo, hi] inside [lambda_1,
lambda_n]: exact extreme eigenvalues for small n (dense generalized eigh),
LOBPCG Ritz values for large n (Ritz values of a symmetric-definite pencil lie
inside its spectrum, so shifts stay in the interior where A - sigma B is
indefinite and pivoting is exercised).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .pencil import Pencil


def spectral_bounds(p: Pencil, maxiter: int = 12, seed: int = 0):
    if p.n <= 3000:
        import scipy.linalg as sla
        w = sla.eigh(p.dense("a"), p.dense("b"), eigvals_only=True)
        return float(w[0]), float(w[-1])
    from scipy.sparse.linalg import lobpcg
    A = p.to_scipy("a").tocsr()
    B = p.to_scipy("b").tocsr()
    rng = np.random.default_rng(seed + 104729)
    X = rng.standard_normal((p.n, 3))
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        lo = lobpcg(A, X, B=B, largest=False, maxiter=maxiter, tol=1e-6)[0]
        hi = lobpcg(A, X, B=B, largest=True, maxiter=maxiter, tol=1e-6)[0]
    return float(np.min(lo)), float(np.max(hi))


def uniform_shifts(lo: float, hi: float, m: int) -> np.ndarray:
    i = np.arange(m, dtype=np.float64)
    return lo + (i + 0.5) * (hi - lo) / m
