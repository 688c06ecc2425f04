"""Tight-binding pencils on jittered lattices — the BASELINE.json configs.

Recipe (BASELINE.json ``configs``; SURVEY.md §8(c) reading 10 fixes the
details BASELINE.json leaves open; DESIGN.md §"Input recipe" restates it):

* atoms on an ``nx x ny x nz`` cubic lattice, spacing 1, lexicographic
  (x slowest) order, each position jittered by U(-j, j)^3 (j = 0.1);
  an axis may be periodic (minimum image), c4 is periodic along z;
* ``o`` orbitals per atom, dof = atom*o + orbital;
* A on-site blocks (M + M^T)/2 with M ~ U(-2, 2)^{o x o};
* B on-site blocks I + 0.05 (U + U^T)/2 with U ~ U(-1, 1)^{o x o};
* every atom pair i < j with distance r <= cutoff couples through
  H_ij = exp(-r) N(0,1)^{o x o} in A (A_ji = H_ij^T) and
  B_ij = 0.05 exp(-r) U(-1,1)^{o x o} in B;
* random draws in this order: positions, A on-site, B on-site, all H_ij
  (pairs in lexicographic (i, j) order), all B_ij;
* B is shifted by c*I only if lambda_min(B) < 0.5, with
  c = ceil((0.5 - lambda_min + 0.01) * 1000) / 1000 (rounded so the stored
  matrix is bit-reproducible across hosts).

The ELSES matrices the paper measured on are not in the
container; these pencils stand in for them.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
from scipy.spatial import cKDTree

from .pencil import Pencil, csc_order

# BASELINE.json configs[0..4] -> c1..c5.  seed = config index.
CONFIGS = {
    1: dict(shape=(5, 5, 10), o=4, cutoff=1.8, periodic=(False, False, False), k_frac=0.3, seed=1),
    2: dict(shape=(20, 20, 20), o=4, cutoff=1.8, periodic=(False, False, False), k_frac=0.3, seed=2),
    3: dict(shape=(30, 30, 30), o=9, cutoff=1.8, periodic=(False, False, False), k_frac=0.25, seed=3),
    4: dict(shape=(10, 10, 3750), o=4, cutoff=1.8, periodic=(False, False, True), k_frac=0.4, seed=4),
    5: dict(shape=(50, 50, 50), o=4, cutoff=2.2, periodic=(False, False, False), k_frac=None, seed=5),
}


def config(index: int, seed: int | None = None, shape=None, **over) -> Pencil:
    """Generate BASELINE.json configs[index-1] (optionally with another seed/shape)."""
    kw = dict(CONFIGS[index])
    if seed is not None:
        kw["seed"] = seed
    if shape is not None:
        kw["shape"] = tuple(shape)
    kw.update(over)
    p = tb_pencil(**kw)
    p.name = f"c{index}" + ("" if shape is None else "-" + "x".join(map(str, shape)))
    return p


def _lambda_min_spd(B: sp.spmatrix, seed: int) -> float:
    n = B.shape[0]
    if n <= 6000:
        return float(np.linalg.eigvalsh(B.toarray())[0])
    from scipy.sparse.linalg import lobpcg
    rng = np.random.default_rng(seed + 7919)
    X = rng.standard_normal((n, 4))
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        vals = lobpcg(B.tocsr(), X, largest=False, tol=1e-5, maxiter=60)[0]
    return float(np.min(vals))


def tb_pencil(shape=(5, 5, 10), o=4, cutoff=1.8, periodic=(False, False, False),
              seed=0, k_frac=None, jitter=0.1, b_min=0.5) -> Pencil:
    nx, ny, nz = shape
    dims = np.array(shape, dtype=np.float64)
    per = np.array(periodic, dtype=bool)
    rng = np.random.default_rng(seed)
    natoms = nx * ny * nz
    n = natoms * o

    grid = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"),
                    axis=-1).reshape(-1, 3).astype(np.float64)
    pos = grid + rng.uniform(-jitter, jitter, size=(natoms, 3))
    Mon = rng.uniform(-2.0, 2.0, size=(natoms, o, o))
    Aon = 0.5 * (Mon + Mon.transpose(0, 2, 1))
    Uon = rng.uniform(-1.0, 1.0, size=(natoms, o, o))
    Bon = np.eye(o)[None] + 0.05 * 0.5 * (Uon + Uon.transpose(0, 2, 1))
    del Mon, Uon

    # neighbour pairs (i < j) within the cutoff, periodic axes by minimum image
    tpos = pos + 1.0
    box = np.where(per, dims, 4.0 * dims + 16.0)
    tpos = np.mod(tpos, box)
    tree = cKDTree(tpos, boxsize=box)
    pairs = tree.query_pairs(cutoff * (1.0 + 1e-9), output_type="ndarray").astype(np.int64)
    d = pos[pairs[:, 1]] - pos[pairs[:, 0]]
    d = np.where(per[None, :], d - dims[None, :] * np.round(d / dims[None, :]), d)
    r = np.sqrt(np.sum(d * d, axis=1))
    keep = r <= cutoff
    pairs, r = pairs[keep], r[keep]
    order = np.lexsort((pairs[:, 1], pairs[:, 0]))
    pairs, r = pairs[order], r[order]
    npairs = pairs.shape[0]
    w = np.exp(-r)
    H = w[:, None, None] * rng.standard_normal(size=(npairs, o, o))
    Bp = 0.05 * w[:, None, None] * rng.uniform(-1.0, 1.0, size=(npairs, o, o))

    # lower-triangle coordinates: on-site (p >= q) and pair blocks (row in atom j)
    pq = np.array([(p, q) for p in range(o) for q in range(o) if p >= q], dtype=np.int64)
    at = np.arange(natoms, dtype=np.int64)
    on_r = (at[:, None] * o + pq[None, :, 0]).ravel()
    on_c = (at[:, None] * o + pq[None, :, 1]).ravel()
    on_a = Aon[:, pq[:, 0], pq[:, 1]].ravel()
    on_b = Bon[:, pq[:, 0], pq[:, 1]].ravel()
    aa, bb = np.meshgrid(np.arange(o), np.arange(o), indexing="ij")   # H[a, b] -> (j*o+b, i*o+a)
    pr_r = (pairs[:, 1:2] * o + bb.ravel()[None, :]).ravel()
    pr_c = (pairs[:, 0:1] * o + aa.ravel()[None, :]).ravel()
    pr_a = H.reshape(npairs, o * o).ravel()
    pr_b = Bp.reshape(npairs, o * o).ravel()
    del H, Bp
    rows = np.concatenate([on_r, pr_r])
    cols = np.concatenate([on_c, pr_c])
    va = np.concatenate([on_a, pr_a])
    vb = np.concatenate([on_b, pr_b])
    del on_r, on_c, pr_r, pr_c, on_a, on_b, pr_a, pr_b
    colptr, rowidx, perm = csc_order(n, rows, cols)
    del rows, cols
    a = va[perm]
    b = vb[perm]
    del va, vb, perm

    # lambda_min(B) and the SPD shift rule
    Bl = sp.csc_matrix((b, rowidx, colptr), shape=(n, n))
    Bfull = Bl + Bl.T - sp.diags(Bl.diagonal())
    lam_min = _lambda_min_spd(Bfull, seed)
    b_shift = 0.0
    if lam_min < b_min:
        b_shift = math.ceil((b_min - lam_min + 0.01) * 1000.0) / 1000.0
        b[colptr[:-1]] += b_shift
    k = None if k_frac is None else int(round(k_frac * n))
    p = Pencil(n=n, colptr=colptr, rowidx=rowidx, a=a, b=b, o=o, coords=pos, k=k,
               name=f"tb{nx}x{ny}x{nz}o{o}",
               meta=dict(shape=tuple(shape), o=o, cutoff=cutoff, periodic=tuple(bool(x) for x in per),
                         seed=seed, npairs=int(npairs), lambda_min_B=lam_min, b_shift=b_shift,
                         jitter=jitter))
    return p
