"""Pins of oracle/lanczos.py (stages 1 and 3) against what the paper and the
mathematics fix: the decomposition identity Eq. (2.1), B-orthonormality,
Ritz-value interlacing, sigma^(1) = Rayleigh quotient
(PAPER.md:248), closed-form spectra of diagonal pencils, LAPACK eigh
(lambda_k to 1e-10), Proposition 2 and Proposition 3
(the bounds Gamma_i contain eigenvalues)."""
import numpy as np
import pytest
import scipy.sparse as sp

import kepgen
import oracle
import oracle.bisection
from oracle.lanczos import LanczosState, lanczos_decomposition, tridiag_eig


def _start(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def _c1():
    p = kepgen.config(1)
    return p.dense("a"), p.dense("b")


def test_lanczos_identity_and_orthonormality():
    A, B = _c1()
    st = lanczos_decomposition(A, B, _start(A.shape[0], 1), 12)
    V = np.array(st.V[:12]).T
    T = np.diag(st.alpha) + np.diag(st.beta[:-1], 1) + np.diag(st.beta[:-1], -1)
    vnext = st.r / st.beta[-1]
    E = A @ V - B @ V @ T - np.outer(B @ vnext, np.eye(12)[-1]) * st.beta[-1]
    assert np.linalg.norm(E) <= 1e-8 * np.linalg.norm(A)
    assert np.allclose(V.T @ B @ V, np.eye(12), atol=1e-12)
    assert abs(vnext @ B @ V).max() < 1e-12


def test_ritz_interlacing_and_rayleigh_start():
    A, B = _c1()
    v0 = _start(A.shape[0], 2)
    st = LanczosState()
    lo, hi = [], []
    for j in range(1, 9):
        lanczos_decomposition(A, B, v0, 1, state=st)
        th = tridiag_eig(st.alpha, st.beta[:-1])[0]
        lo.append(th[0]); hi.append(th[-1])
    assert np.isclose(lo[0], v0 @ A @ v0 / (v0 @ B @ v0), rtol=1e-13)          # theta_1^(1)
    assert all(np.diff(lo) < 0) and all(np.diff(hi) > 0)                          # monotone (interlacing)
    w = oracle.eigvals_pencil(A, B)
    assert lo[-1] > w[0] and hi[-1] < w[-1]


def test_alg2_diagonal_pencil_closed_form():
    n, k = 64, 32
    A = np.diag(np.arange(1.0, n + 1))
    B = np.eye(n)
    nu = lambda s: int(np.sum(np.arange(1.0, n + 1) < s))
    lo, hi, nl, nh, j, trace = oracle.initial_interval_alg2(A, B, k, _start(n, 3), nu)
    assert nl < k <= nh and nl == nu(lo) and nh == nu(hi)
    assert lo <= k < hi                                                            # lambda_k = k
    assert np.isclose(trace[0][0], np.average(np.arange(1.0, n + 1), weights=_start(n, 3) ** 2))


@pytest.mark.parametrize("k", [1, 300, 700, 1000])
def test_alg2_c1_brackets_lambda_k(k):
    A, B = _c1()
    w = oracle.eigvals_pencil(A, B)
    nu = lambda s: oracle.nu_eig(A, B, s, eigvals=w)
    lo, hi, nl, nh, j, _ = oracle.initial_interval_alg2(A, B, k, _start(A.shape[0], 4), nu)
    assert nl < k <= nh and lo <= w[k - 1] < hi
    if 1 < k < A.shape[0]:
        assert j <= 12          # interior k: a few steps (the paper saw j = 2)


def test_alg3_c1_lambda_k_and_bounds():
    A, B = _c1()
    w = oracle.eigvals_pencil(A, B)
    k = 300
    nu = lambda s: oracle.nu_eig(A, B, s, eigvals=w)
    lo, hi, nl, nh, _, _ = oracle.initial_interval_alg2(A, B, k, _start(A.shape[0], 5), nu)
    (lo, hi, nl, nh), _, _ = oracle.bisection.bisect_alg1p(nu, k, lo, hi, nl, nh, m_max=20)
    res = oracle.si_lanczos_alg3(A, B, k, lo, hi, nl, nh, _start(A.shape[0], 6))
    assert abs(res.lam - w[k - 1]) <= 1e-10 * abs(w[k - 1])
    # Prop. 3: each bound contains an eigenvalue (here: the one with the same index)
    m = nh - nl
    wi = w[nl:nh]
    assert np.all(np.abs(res.lams - wi) <= res.etas + 1e-13 * np.abs(wi))     # bound + rounding of both sides
    x = res.x
    assert np.linalg.norm(A @ x - res.lam * (B @ x)) / np.linalg.norm(x) < 1e-10


def test_alg3_diagonal_pencil_exact():
    n = 40
    d = np.arange(1.0, n + 1) ** 1.5
    A, B = np.diag(d), np.diag(np.linspace(1.0, 2.0, n))
    lam = np.sort(d / np.linspace(1.0, 2.0, n))
    k = 17
    nu = lambda s: int(np.sum(lam < s))
    lo, hi = lam[k - 3] + 1e-3, lam[k + 1] + 1e-3         # 3 eigenvalues inside (k-1, k, k+1 .. )
    res = oracle.si_lanczos_alg3(A, B, k, lo, hi, nu(lo), nu(hi), _start(n, 8))
    assert abs(res.lam - lam[k - 1]) <= 1e-12 * lam[k - 1]


def test_prop2_orthogonality_formula():
    A, B = _c1()
    n = A.shape[0]
    sigma = 0.1
    M = np.linalg.solve(A - sigma * B, B)                 # (A - sigma B)^-1 B
    w = _start(n, 9)
    w = w / np.sqrt(w @ B @ w)
    W, alpha, beta = [w], [], []
    for j in range(8):
        z = M @ W[-1]
        a = W[-1] @ B @ z
        r = z - a * W[-1] - (beta[-1] * W[-2] if j else 0)
        for _ in range(2):
            r = r - np.array(W).T @ (np.array(W) @ (B @ r))
        b = np.sqrt(r @ B @ r)
        alpha.append(a); beta.append(b)
        W.append(r / b)
    th, Y = tridiag_eig(alpha, beta[:-1])
    Wm = np.array(W[:8]).T
    X = Wm @ Y * th + np.outer(W[8] * beta[-1], Y[-1])
    g = beta[-1] * Y[-1] / th
    for l_, m_ in [(0, 1), (2, 7), (3, 5)]:
        lhs = abs(X[:, l_] @ B @ X[:, m_]) / np.sqrt(X[:, l_] @ B @ X[:, l_]) / np.sqrt(X[:, m_] @ B @ X[:, m_])
        rhs = abs(g[l_]) / np.sqrt(1 + g[l_] ** 2) * abs(g[m_]) / np.sqrt(1 + g[m_] ** 2)
        assert np.isclose(lhs, rhs, rtol=1e-6, atol=1e-14)
