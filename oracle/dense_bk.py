"""Textbook Bunch-Kaufman LDL^T and the inertia of D (O-dense).

Follows Alg. 1 lines 3-4: L D L^T <- P(A - sigma B)P^T,
nu := nu_0(D, I), with P the Bunch-Kaufman stability permutation the paper
cites ([BunchKaufman1977]); D is block diagonal with 1x1 and 2x2
blocks.  The pivot rule is the classical one (LAPACK dsytf2, lower), written
step by step:

  alpha = (1 + sqrt(17)) / 8
  colmax = max_{i>k} |s_ik|  (row imax; ties -> lowest index)
  if max(|s_kk|, colmax) == 0 : zero pivot (singular), nothing to update
  elif |s_kk| >= alpha colmax : 1x1 at k
  else rowmax = max_{j != imax} |s_imax,j| over the active block
       if |s_kk| rowmax >= alpha colmax^2        : 1x1 at k
       elif |s_imax,imax| >= alpha rowmax        : 1x1 at imax (swap k <-> imax)
       else                                      : 2x2 on {k, imax} (swap k+1 <-> imax)

Inertia of D (reading R2): 1x1 by sign;
2x2 [d11 d21; d21 d22] by sign(det) computed in the scaled form
(d11/d21)(d22/d21) - 1:  det < 0 -> one negative, one positive;
det > 0 -> two of the sign of d11; det == 0 -> one zero plus sign(trace).

Plain numpy, fp64, full symmetric storage, physical row/column swaps.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

ALPHA = (1.0 + math.sqrt(17.0)) / 8.0
TAU_SING = 1e-14          # SPEC.md:158 breakdown threshold, relative to max|S|


@dataclass
class Inertia:
    n_neg: int = 0
    n_zero: int = 0
    n_pos: int = 0
    n_2x2: int = 0
    n_delayed: int = 0            # sparse oracle only
    min_abs_pivot: float = math.inf
    smax: float = 0.0             # max |s_ij| of the matrix factored
    factors: dict = field(default_factory=dict)

    @property
    def singular(self) -> bool:
        return self.n_zero > 0 or self.min_abs_pivot <= TAU_SING * self.smax

    def add(self, other: "Inertia") -> None:
        self.n_neg += other.n_neg
        self.n_zero += other.n_zero
        self.n_pos += other.n_pos
        self.n_2x2 += other.n_2x2
        self.n_delayed += other.n_delayed
        self.min_abs_pivot = min(self.min_abs_pivot, other.min_abs_pivot)


def block_inertia_1x1(d: float):
    """(neg, zero, pos, min|eig|) of a 1x1 pivot."""
    if d < 0.0:
        return 1, 0, 0, -d
    if d > 0.0:
        return 0, 0, 1, d
    return 0, 1, 0, 0.0


def block_inertia_2x2(d11: float, d21: float, d22: float):
    """(neg, zero, pos, min|eig|) of the symmetric 2x2 block [d11 d21; d21 d22]."""
    if d21 == 0.0:
        a = block_inertia_1x1(d11)
        b = block_inertia_1x1(d22)
        return a[0] + b[0], a[1] + b[1], a[2] + b[2], min(a[3], b[3])
    t = (d11 / d21) * (d22 / d21) - 1.0          # det / d21^2, LAPACK dsytf2 scaling
    ev = np.linalg.eigvalsh(np.array([[d11, d21], [d21, d22]]))
    mn = float(np.min(np.abs(ev)))
    if t < 0.0:
        return 1, 0, 1, mn
    if t > 0.0:
        return (2, 0, 0, mn) if d11 < 0.0 else (0, 0, 2, mn)
    tr = d11 + d22
    return (1 if tr < 0 else 0), 1, (1 if tr > 0 else 0), 0.0


def _swap(S: np.ndarray, i: int, j: int, perm: np.ndarray) -> None:
    if i == j:
        return
    S[[i, j], :] = S[[j, i], :]
    S[:, [i, j]] = S[:, [j, i]]
    perm[[i, j]] = perm[[j, i]]


def bk_ldl(S: np.ndarray, return_factors: bool = False) -> Inertia:
    """Bunch-Kaufman LDL^T of the dense symmetric S; returns the inertia of D.

    With ``return_factors`` the result carries L (unit lower), D (block
    diagonal) and perm such that S[perm][:, perm] = L D L^T.
    """
    S = np.array(S, dtype=np.float64, copy=True)
    n = S.shape[0]
    res = Inertia(smax=float(np.max(np.abs(S))) if n else 0.0)
    perm = np.arange(n)
    L = np.eye(n) if return_factors else None
    D = np.zeros((n, n)) if return_factors else None
    k = 0
    while k < n:
        absakk = abs(S[k, k])
        if k < n - 1:
            col = np.abs(S[k + 1:, k])
            imax = k + 1 + int(np.argmax(col))
            colmax = float(col[imax - k - 1])
        else:
            imax, colmax = k, 0.0
        if max(absakk, colmax) == 0.0:
            # zero column: zero pivot, singular (LAPACK sets info and moves on)
            res.n_zero += 1
            res.min_abs_pivot = 0.0
            k += 1
            continue
        kstep, kp = 1, k
        if absakk < ALPHA * colmax:
            row = np.concatenate([np.abs(S[imax, k:imax]), np.abs(S[imax + 1:, imax])])
            rowmax = float(np.max(row))
            if absakk * rowmax >= ALPHA * colmax * colmax:
                kp = k
            elif abs(S[imax, imax]) >= ALPHA * rowmax:
                kp = imax
            else:
                kp, kstep = imax, 2
        kk = k + kstep - 1
        _swap(S, kk, kp, perm)
        if return_factors and kk != kp:
            L[[kk, kp], :k] = L[[kp, kk], :k]
        if kstep == 1:
            d = S[k, k]
            v = S[k + 1:, k].copy()
            S[k + 1:, k + 1:] -= np.outer(v, v) / d
            neg, zer, pos, mn = block_inertia_1x1(d)
            if return_factors:
                L[k + 1:, k] = v / d
                D[k, k] = d
        else:
            Dk = S[k:k + 2, k:k + 2].copy()
            V = S[k + 2:, k:k + 2].copy()
            W = V @ np.linalg.inv(Dk)
            S[k + 2:, k + 2:] -= W @ V.T
            neg, zer, pos, mn = block_inertia_2x2(Dk[0, 0], Dk[1, 0], Dk[1, 1])
            res.n_2x2 += 1
            if return_factors:
                L[k + 2:, k:k + 2] = W
                D[k:k + 2, k:k + 2] = Dk
        res.n_neg += neg
        res.n_zero += zer
        res.n_pos += pos
        res.min_abs_pivot = min(res.min_abs_pivot, mn)
        k += kstep
    if return_factors:
        res.factors = dict(L=L, D=D, perm=perm)
    return res


def reconstruct(S: np.ndarray, inertia: Inertia) -> float:
    """||P S P^T - L D L^T||_F / ||S||_F for factors returned by bk_ldl."""
    f = inertia.factors
    p = f["perm"]
    R = S[np.ix_(p, p)] - f["L"] @ f["D"] @ f["L"].T
    return float(np.linalg.norm(R) / np.linalg.norm(S))


def nu_dense(A: np.ndarray, B: np.ndarray, sigma: float) -> Inertia:
    """Inertia of D for S = A - sigma B (Alg. 1 lines 3-4); nu = .n_neg."""
    return bk_ldl(np.asarray(A) - sigma * np.asarray(B))
