"""Brute-force symbolic factorisation (SPEC.md:59-76 symbolic_factorize; pin P9).

Simulates Gaussian elimination on a dense boolean matrix of the permuted
pattern: eliminating column j makes every pair of its remaining nonzero rows
adjacent (fill).  Gives, for the ordering supplied, the nonzero count of every
column of L (diagonal included) and the elimination tree
(parent(j) = min{i > j : l_ij != 0}).  O(n^3) booleans: tiny n only.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np


def brute_symbolic(n: int, colptr, rowidx, position):
    """``position[i]`` = place of original index i in the elimination order."""
    M = np.zeros((n, n), dtype=bool)
    col = np.repeat(np.arange(n), np.diff(colptr))
    r = np.asarray(position)[np.asarray(rowidx)]
    c = np.asarray(position)[col]
    M[r, c] = True
    M[c, r] = True
    np.fill_diagonal(M, True)
    counts = np.zeros(n, dtype=np.int64)
    parent = np.full(n, -1, dtype=np.int64)
    for j in range(n):
        rows = np.nonzero(M[j + 1:, j])[0] + j + 1
        counts[j] = rows.shape[0] + 1
        if rows.shape[0]:
            parent[j] = rows[0]
            M[np.ix_(rows, rows)] = True
    return counts, parent


def factor_flops(counts) -> int:
    """Algorithmic LDL^T flops of a column-count vector:
    eliminating a column with m = c_j - 1 sub-diagonal entries costs m
    divisions plus a symmetric rank-1 update of m(m+1)/2 lower entries at one
    multiply-add (2 flops) each, i.e. m^2 + 2m; summed over all columns."""
    m = np.asarray(counts, dtype=np.int64) - 1
    return int(np.sum(m * m + 2 * m))
