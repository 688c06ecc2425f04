"""Closed-form spectra used as pins.

Twin pencils (kepgen.twin): A = M_A (x) H + I (x) E, B = I + M_B (x) G with
H, E, G = Q diag(h|e|g) Q^T and M_* polynomials in commuting 1-D lattice
operators T_ax.  In the common eigenbasis (lattice modes (x) columns of Q)
both A and B are diagonal, so every eigenvalue of the pencil is

    lambda(theta, p) = (e_p + h_p mu_A(theta)) / (1 + g_p mu_B(theta)),
    mu(theta) = prod_ax (1 + t_ax tau_ax) - 1 + u sum_ax (tau_ax^2 - 2),

with tau = 2 cos(pi j / (N + 1)), j = 1..N on an open axis and
tau = 2 cos(2 pi j / N), j = 0..N-1 on a periodic axis (eigenvalues of the
tridiagonal / circulant T with unit off-diagonals).

Sturm count (P5): for a symmetric tridiagonal T (B = I) the number of
eigenvalues below sigma is the number of negative q_i in
q_1 = a_1 - sigma, q_i = (a_i - sigma) - b_{i-1}^2 / q_{i-1}
(the unpivoted LDL^T recurrence; Givens' bisection).
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np


def _tau(N: int, periodic: bool) -> np.ndarray:
    if periodic:
        return 2.0 * np.cos(2.0 * np.pi * np.arange(N) / N)
    if N == 1:
        return np.zeros(1)
    return 2.0 * np.cos(np.pi * np.arange(1, N + 1) / (N + 1))


def _mu(shape, periodic, t, u) -> np.ndarray:
    taus = [_tau(N, p) for N, p in zip(shape, periodic)]
    tx, ty, tz = np.meshgrid(*taus, indexing="ij")
    prod = (1 + t[0] * tx) * (1 + t[1] * ty) * (1 + t[2] * tz) - 1.0
    return (prod + u * ((tx ** 2 - 2) + (ty ** 2 - 2) + (tz ** 2 - 2))).ravel()


def twin_eigenvalues(meta: dict) -> np.ndarray:
    """All n eigenvalues of a twin pencil, ascending (meta = Pencil.meta['twin'])."""
    muA = _mu(meta["shape"], meta["periodic"], meta["tA"], meta["uA"])
    muB = _mu(meta["shape"], meta["periodic"], meta["tB"], meta["uB"])
    h, e, g = (np.asarray(meta[x]) for x in ("h", "e", "g"))
    lam = (e[None, :] + h[None, :] * muA[:, None]) / (1.0 + g[None, :] * muB[:, None])
    return np.sort(lam.ravel())


def nu_twin(meta: dict, sigma, eigvals=None):
    w = twin_eigenvalues(meta) if eigvals is None else eigvals
    s = np.asarray(sigma, dtype=np.float64)
    r = np.searchsorted(w, s, side="left")
    return r if s.ndim else int(r)


def sturm_count(diag: np.ndarray, off: np.ndarray, sigma: float) -> int:
    """#eigenvalues < sigma of the symmetric tridiagonal (diag, off)."""
    count = 0
    q = 1.0
    for i in range(diag.shape[0]):
        b2 = off[i - 1] ** 2 if i > 0 else 0.0
        q = (diag[i] - sigma) - (b2 / q if i > 0 else 0.0)
        if q == 0.0:
            q = -1e-300           # sigma exactly at a pivot breakdown: perturb (Kahan)
        if q < 0.0:
            count += 1
    return count
