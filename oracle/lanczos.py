"""Stages 1 and 3 of the three-stage k-th eigenpair method, step by step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain numpy/scipy: the
matrices are scipy sparse (full symmetric) or dense arrays; linear solves use a
library LU (scipy splu / numpy solve) as a step.

- ``lanczos_decomposition``  the j-step Lanczos decomposition Eq. (2.1),
  A V_j = B V_j T_j + B v_{j+1} beta_j e_j^T, V_j B-orthonormal
  (§2.2), full reorthogonalisation in the B-inner product
  (reading R13).
- ``initial_interval_alg2``  Algorithm 2 (§3.1): Ritz values
  theta_1^(j) (k <= nu^(j-1)) or theta_j^(j) (otherwise) as shifts until two
  consecutive shifts bracket lambda_k.
- ``si_lanczos_alg3``        Algorithm 3 (§3.2): SI Lanczos
  Eq. (2.4) with reorthogonalisation at the interval
  midpoint, eigenpairs (2.5) / x_{i,2} (2.7), error bounds
  Eq. (3.1), tests (3.3)-(3.5).

The SI decomposition (A - sigma B)^-1 V~ = B^-1 V~ T~ + B^-1 v~_{j+1} beta~ e_j^T
is run on the companions w = B^-1 v~ (B-orthonormal): (A - sigma B)^-1 B W =
W T~ + w_{j+1} beta~ e_j^T, which needs one solve with A - sigma B and one
product with B per step and no solve with B.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def _mv(M, x):
    return M @ x


def _factor(M):
    if sp.issparse(M):
        lu = spla.splu(sp.csc_matrix(M))
        return lu.solve
    lu = sla.lu_factor(np.asarray(M))
    return lambda b: sla.lu_solve(lu, b)


def tridiag_eig(alpha, beta):
    """Eigenpairs of the symmetric tridiagonal T (diagonal alpha, off-diagonal beta), ascending."""
    alpha = np.asarray(alpha, float)
    beta = np.asarray(beta, float)
    if len(alpha) == 1:
        return alpha.copy(), np.ones((1, 1))
    return sla.eigh_tridiagonal(alpha, beta)


@dataclass
class LanczosState:
    V: list = field(default_factory=list)      # B-orthonormal basis v_1..v_j
    U: list = field(default_factory=list)      # u_i = B v_i
    alpha: list = field(default_factory=list)
    beta: list = field(default_factory=list)   # beta_1..beta_j (beta_j scales v_{j+1})
    r: np.ndarray = None                        # unnormalised v_{j+1} beta_j
    rhat: np.ndarray = None                     # B r


def lanczos_decomposition(A, B, v0, steps, solve_B=None, state=None):
    """Extend the Lanczos decomposition Eq. (2.1) by `steps` steps."""
    solve_B = solve_B or _factor(B)
    st = state or LanczosState()
    if not st.V:
        v = np.asarray(v0, float)
        v = v / np.sqrt(v @ _mv(B, v))
        st.V.append(v)
        st.U.append(_mv(B, v))
    for _ in range(steps):
        j = len(st.alpha)
        if j == len(st.V):                      # v_{j+1} pending from the previous step
            st.V.append(st.r / st.beta[-1])
            st.U.append(st.rhat / st.beta[-1])
        v, u = st.V[j], st.U[j]
        w = _mv(A, v)                           # A v_j
        a = float(v @ w)
        rh = w - a * u
        if j > 0:
            rh = rh - st.beta[-1] * st.U[j - 1]
        for _ in range(2):                      # full reorthogonalisation: rh -= U (V^T rh)
            Vm = np.array(st.V)
            Um = np.array(st.U)
            rh = rh - Um.T @ (Vm @ rh)
        r = solve_B(rh)                         # B^-1 (A v_j - ...)
        b = float(np.sqrt(max(rh @ r, 0.0)))
        st.alpha.append(a)
        st.beta.append(b)
        st.r, st.rhat = r, rh
    return st


def initial_interval_alg2(A, B, k, v0, nu, jmax=200):
    """Algorithm 2 -> (sigma_l, sigma_u, nu_l, nu_u, j, trace)."""
    solve_B = _factor(B)
    st = LanczosState()
    nu_prev = 0                                 # nu^(0) := 0
    sig_prev = None
    trace = []
    for j in range(1, jmax + 1):
        lanczos_decomposition(A, B, v0, 1, solve_B, st)              # j-step decomposition
        theta = tridiag_eig(st.alpha, st.beta[:-1])[0]               # Eq. (2.2)
        sig = theta[0] if k <= nu_prev else theta[-1]
        v = nu(sig)
        trace.append((sig, v))
        if j != 1 and (v < k <= nu_prev or nu_prev < k <= v):
            lo, hi = min(sig_prev, sig), max(sig_prev, sig)
            return lo, hi, min(nu_prev, v), max(nu_prev, v), j, trace
        nu_prev, sig_prev = v, sig
    raise RuntimeError("Algorithm 2 did not bracket lambda_k")


@dataclass
class SiResult:
    lam: float
    x: np.ndarray
    j: int
    eta: float
    relres: float
    reldiff: float
    lams: np.ndarray        # the m eigenvalues of the interval, ascending
    etas: np.ndarray
    sigma: float


def si_lanczos_alg3(A, B, k, lo, hi, nu_lo, nu_hi, v0, tau_res=1e-10, tau_diff=1e-10, jmax=500):
    """Algorithm 3."""
    l = k - nu_lo                               # 1-based index inside the interval
    m = nu_hi - nu_lo
    sigma = (lo + hi) / 2.0
    solve = _factor(A - sigma * B)
    w = np.asarray(v0, float)
    w = w / np.sqrt(w @ _mv(B, w))              # v~_1 / ||v~_1||_{B^-1}  <=>  w_1 B-normalised
    W, Vt = [w], [_mv(B, w)]
    alpha, beta = [], []
    prev = None
    for j in range(1, jmax + 1):
        z = solve(Vt[-1])                       # (A - sigma B)^-1 v~_j
        a = float(Vt[-1] @ z)
        r = z - a * W[-1]
        if j > 1:
            r = r - beta[-1] * W[-2]
        for _ in range(2):                      # reorthogonalisation in the B-inner product
            r = r - np.array(W).T @ (np.array(Vt) @ r)
        u = _mv(B, r)
        b = float(np.sqrt(max(r @ u, 0.0)))
        alpha.append(a)
        beta.append(b)
        if j >= m:
            th, Y = tridiag_eig(alpha, beta[:-1])                    # Eq. (2.5)
            order = np.argsort(-np.abs(th), kind="stable")           # |theta~_1| >= |theta~_2| >= ...
            th, Y = th[order], Y[:, order]
            Wm = np.array(W).T
            lam = sigma + 1.0 / th                                   # Eq. (2.6)
            X = Wm @ Y * th + np.outer(r, Y[-1, :])                  # x_{i,2} = theta W y + w_{j+1} beta (e_j^T y)
            rho = np.abs(b * Y[-1, :] / th)
            eta = rho / np.abs(th) / np.sqrt(1.0 + rho ** 2)         # Eq. (3.1)
            lm, em, Xm = lam[:m], eta[:m], X[:, :m]
            inc = bool(np.all(lm - em >= lo) and np.all(lm + em < hi))          # (3.3)
            srt = np.argsort(lm)
            dis = bool(np.all(lm[srt][:-1] + em[srt][:-1] < lm[srt][1:] - em[srt][1:]))   # (3.4)
            res = np.array([np.linalg.norm(_mv(A, Xm[:, i]) - lm[i] * _mv(B, Xm[:, i])) / np.linalg.norm(Xm[:, i])
                            for i in range(m)])
            dif = np.full(m, np.inf)
            if prev is not None:                                      # Eq. (3.5), sign-aligned, equal 2-norms
                for i in range(m):
                    xp = prev[:, i]
                    xc = Xm[:, i] * (np.linalg.norm(xp) / np.linalg.norm(Xm[:, i]))
                    if xc @ xp < 0:
                        xc = -xc
                    dif[i] = np.linalg.norm(xc - xp) / np.linalg.norm(xp)
            prev = Xm.copy()
            if inc and dis and np.all(res < tau_res) and np.all(dif < tau_diff):
                o2 = np.argsort(lm)                                   # back to increasing order
                i = o2[l - 1]
                return SiResult(lam=float(lm[i]), x=Xm[:, i], j=j, eta=float(em[i]), relres=float(res[i]),
                                reldiff=float(dif[i]), lams=lm[o2], etas=em[o2], sigma=sigma)
        W.append(r / b)
        Vt.append(u / b)
    raise RuntimeError("Algorithm 3 did not converge")
