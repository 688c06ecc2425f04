"""Separable lattice "twin" pencils (SURVEY.md §8(c) pin P4).

A = M_A (x) H + I (x) E,      B = I + M_B (x) G,

with lattice operators built from commuting 1-D tridiagonal (open axis) or
circulant (periodic axis) matrices T_x, T_y, T_z (ones on the off-diagonals):

M = (I + t_x T_x) (x) (I + t_y T_y) (x) (I + t_z T_z) - I + u * sum_ax (T_ax^2 - 2I)

(x slowest, matching the atom order of :mod:`kepgen.tb`), and o x o orbital
blocks H = Q diag(h) Q^T, E = Q diag(e) Q^T, G = Q diag(g) Q^T sharing one
random orthogonal Q.  The block pattern is exactly the 27-point (u = 0) or
27+6-point (u != 0) stencil, i.e. the neighbour-block pattern of the
cutoff-1.8 (resp. cutoff-2.2-like) tight-binding configs, with dense o x o
blocks.  The generator only draws parameters and assembles the matrices;
the closed-form spectrum lives in ``oracle/closed_form.py`` and is computed
from ``Pencil.meta['twin']``.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .pencil import Pencil, csc_order


def _T(N: int, periodic: bool) -> sp.csr_matrix:
    if periodic:
        assert N >= 3, "periodic axis needs N >= 3"
        i = np.arange(N)
        rows = np.concatenate([i, i])
        cols = np.concatenate([(i + 1) % N, (i - 1) % N])
        return sp.csr_matrix((np.ones(2 * N), (rows, cols)), shape=(N, N))
    if N == 1:
        return sp.csr_matrix((1, 1))
    return sp.diags([np.ones(N - 1), np.ones(N - 1)], [-1, 1], format="csr")


def _kron3(X, Y, Z):
    return sp.kron(sp.kron(X, Y, format="csr"), Z, format="csr")


def _lattice_operator(shape, periodic, t, u):
    Ts = [_T(N, p) for N, p in zip(shape, periodic)]
    Is = [sp.identity(N, format="csr") for N in shape]
    F = [Is[a] + t[a] * Ts[a] for a in range(3)]
    M = _kron3(F[0], F[1], F[2]) - sp.identity(int(np.prod(shape)), format="csr")
    if u != 0.0:
        for a in range(3):
            W = [Is[0], Is[1], Is[2]]
            W[a] = (Ts[a] @ Ts[a] - 2.0 * Is[a]).tocsr()
            M = M + u * _kron3(W[0], W[1], W[2])
    return M.tocsr()


def twin_pencil(shape=(5, 5, 10), o=4, periodic=(False, False, False), seed=100,
                tA=(0.5, 0.5, 0.5), tB=(0.05, 0.05, 0.05), uA=0.0, uB=0.0,
                k_frac=None) -> Pencil:
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((o, o)))
    h = rng.standard_normal(o)
    e = rng.uniform(-2.0, 2.0, o)
    g = rng.uniform(-1.0, 1.0, o)
    H = (Q * h) @ Q.T
    E = (Q * e) @ Q.T
    G = (Q * g) @ Q.T
    H = 0.5 * (H + H.T)
    E = 0.5 * (E + E.T)
    G = 0.5 * (G + G.T)
    MA = _lattice_operator(shape, periodic, tA, uA)
    MB = _lattice_operator(shape, periodic, tB, uB)
    natoms = int(np.prod(shape))
    n = natoms * o
    # block pattern (lower, I >= J) and the lattice-operator value of every block
    P = (abs(MA) + abs(MB) + sp.identity(natoms, format="csr")).tocoo()
    low = P.row >= P.col
    BI = P.row[low].astype(np.int64)
    BJ = P.col[low].astype(np.int64)

    def lookup(M):
        M = M.tocoo()
        key = M.row.astype(np.int64) * natoms + M.col
        order = np.argsort(key)
        key, val = key[order], M.data[order]
        q = BI * natoms + BJ
        pos = np.searchsorted(key, q)
        pos = np.minimum(pos, key.shape[0] - 1)
        hit = key[pos] == q
        return np.where(hit, val[pos], 0.0)

    mA = lookup(MA)
    mB = lookup(MB)
    diag = BI == BJ
    pp, qq = np.meshgrid(np.arange(o), np.arange(o), indexing="ij")
    pp, qq = pp.ravel(), qq.ravel()
    rows = (BI[:, None] * o + pp[None, :]).ravel()
    cols = (BJ[:, None] * o + qq[None, :]).ravel()
    va = (mA[:, None] * H[pp, qq][None, :] + diag[:, None] * E[pp, qq][None, :]).ravel()
    vb = (diag[:, None] * (pp == qq)[None, :] + mB[:, None] * G[pp, qq][None, :]).ravel()
    keep = rows >= cols
    rows, cols, va, vb = rows[keep], cols[keep], va[keep], vb[keep]
    colptr, rowidx, perm = csc_order(n, rows, cols)
    a = va[perm]
    b = vb[perm].astype(np.float64)
    grid = np.stack(np.meshgrid(*[np.arange(N) for N in shape], indexing="ij"), axis=-1)
    coords = grid.reshape(-1, 3).astype(np.float64)
    k = None if k_frac is None else int(round(k_frac * n))
    return Pencil(n=n, colptr=colptr, rowidx=rowidx, a=a, b=b, o=o,
                  coords=coords, k=k, name="twin" + "x".join(map(str, shape)) + f"o{o}",
                  meta=dict(twin=dict(shape=tuple(shape), periodic=tuple(periodic), tA=tuple(tA),
                                      tB=tuple(tB), uA=uA, uB=uB, h=h, e=e, g=g), seed=seed))
