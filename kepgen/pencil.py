"""Pencil container and storage helpers (no method arithmetic)."""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import scipy.sparse as sp


@dataclass
class Pencil:
    """A real symmetric / SPD pencil (A, B) on one union sparsity pattern.

    Storage: lower triangle (row >= col), compressed sparse column, 0-based,
    row indices sorted within each column, diagonal always present
    (SPEC.md:22-28 SparseSymmetric; "#nz ... in their lower
    triangular part").  ``a`` and ``b`` are aligned with ``rowidx``.
    """

    n: int
    colptr: np.ndarray          # int64 [n+1]
    rowidx: np.ndarray          # int32 [nnz_lower]
    a: np.ndarray               # float64 [nnz_lower]
    b: np.ndarray               # float64 [nnz_lower]
    o: int = 1                  # dofs (orbitals) per atom; dof = atom*o + orbital
    coords: Optional[np.ndarray] = None   # float64 [natoms, 3] atom positions
    k: Optional[int] = None     # target index k (1-based)
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.rowidx.shape[0])

    @property
    def natoms(self) -> int:
        return self.n // self.o

    def colidx(self) -> np.ndarray:
        """Column index of every stored entry (int64)."""
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.colptr))

    def to_scipy(self, which: str = "a") -> sp.csc_matrix:
        """Full symmetric scipy matrix of A or B (storage expansion only)."""
        vals = self.a if which == "a" else self.b
        L = sp.csc_matrix((vals, self.rowidx, self.colptr), shape=(self.n, self.n))
        D = sp.diags(L.diagonal())
        return (L + L.T - D).tocsc()

    def dense(self, which: str = "a") -> np.ndarray:
        return self.to_scipy(which).toarray()

    def check(self) -> None:
        """Validate the storage invariants of SPEC.md:22-28."""
        n = self.n
        cp, ri = self.colptr, self.rowidx
        assert cp.dtype == np.int64 and ri.dtype == np.int32
        assert cp.shape == (n + 1,) and cp[0] == 0 and cp[-1] == ri.shape[0]
        assert self.a.shape == ri.shape and self.b.shape == ri.shape
        col = self.colidx()
        assert np.all(ri >= col), "entries must be in the lower triangle"
        assert np.all(ri < n)
        # sorted, unique within a column, diagonal first
        same = col[1:] == col[:-1]
        assert np.all(ri[1:][same] > ri[:-1][same]), "rows sorted & unique per column"
        assert np.all(ri[cp[:-1]] == np.arange(n)), "diagonal present"


def lower_csc_from_coo(n, rows, cols, va, vb):
    """Lower CSC (sorted, duplicates summed) from coordinate triples with row>=col."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    assert np.all(rows >= cols)
    order = np.lexsort((rows, cols))
    rows, cols = rows[order], cols[order]
    va = np.asarray(va, dtype=np.float64)[order]
    vb = np.asarray(vb, dtype=np.float64)[order]
    key = cols * n + rows
    uniq = np.ones(key.shape[0], dtype=bool)
    uniq[1:] = key[1:] != key[:-1]
    if not np.all(uniq):
        grp = np.cumsum(uniq) - 1
        va = np.bincount(grp, weights=va)
        vb = np.bincount(grp, weights=vb)
        rows, cols = rows[uniq], cols[uniq]
    colptr = np.zeros(n + 1, dtype=np.int64)
    colptr[1:] = np.cumsum(np.bincount(cols, minlength=n))
    return colptr, rows.astype(np.int32), va, vb


def csc_order(n, rows, cols):
    """Counting-sort coordinates (row >= col, no duplicates) into lower CSC.

    Returns (colptr int64, rowidx int32, perm) with entry e of the CSC equal to
    coordinate perm[e]."""
    nnz = rows.shape[0]
    idx = sp.coo_matrix((np.arange(1, nnz + 1, dtype=np.float64), (rows, cols)), shape=(n, n)).tocsc()
    idx.sort_indices()
    assert idx.nnz == nnz, "duplicate coordinates"
    return idx.indptr.astype(np.int64), idx.indices.astype(np.int32), idx.data.astype(np.int64) - 1


def full_from_lower(n, colptr, rowidx, vals) -> np.ndarray:
    """Dense symmetric matrix from lower CSC (storage expansion only)."""
    L = sp.csc_matrix((vals, rowidx, colptr), shape=(n, n)).toarray()
    return L + L.T - np.diag(np.diag(L))
