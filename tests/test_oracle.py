"""Pins for the oracle.  CPU only.

Each test pins the oracle to something other than itself: LAPACK eigenvalues
(P1), LAPACK's own Bunch-Kaufman (P2), O-dense vs O-sparse (P3), closed-form
twin spectra (P4), Sturm counts (P5), metamorphic identities (P6), the SPEC
worked examples (P7), factor residuals (P8), brute-force symbolic counts (P9).
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg as sla

import kepgen
import oracle
from oracle.bisection import bisect_alg1, bisect_alg1p
from oracle.closed_form import sturm_count
from oracle.dense_bk import block_inertia_2x2, bk_ldl, reconstruct
from oracle.symbolic import brute_symbolic

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


def _rand_sym(rng, n, zero_diag=False):
    M = rng.standard_normal((n, n))
    S = M + M.T
    if zero_diag:
        np.fill_diagonal(S, 0.0)
    return S


def _rand_pencil(rng, n):
    # SPEC.md:485 acceptance 1: B = M^T M + n I
    A = _rand_sym(rng, n)
    M = rng.standard_normal((n, n))
    B = M.T @ M + n * np.eye(n)
    return A, B


# ---------------------------------------------------------------- P7 SPEC worked examples
def test_spec_examples_inertia():
    g = json.load(open(GOLD))
    for case in g["inertia"]:
        r = bk_ldl(np.array(case["S"], dtype=float))
        assert (r.n_neg, r.n_zero, r.n_pos, r.n_2x2) == (case["neg"], case["zero"], case["pos"], case["n2x2"]), case["cite"]


def test_spec_examples_nu():
    g = json.load(open(GOLD))
    for case in g["nu"]:
        A = np.diag(np.array(case["A_diag"], float))
        B = np.diag(np.array(case["B_diag"], float))
        assert oracle.nu_dense(A, B, case["sigma"]).n_neg == case["nu"], case["cite"]
        assert oracle.nu_eig(A, B, case["sigma"]) == case["nu"], case["cite"]


def test_spec_bisection_iterations():
    g = json.load(open(GOLD))["bisection"][0]
    A = np.diag(np.arange(1, g["n"] + 1, dtype=float))
    B = np.eye(g["n"])
    lam, it, _ = bisect_alg1(lambda s: oracle.nu_dense(A, B, s).n_neg, g["k"], g["lo"], g["hi"], g["tau"])
    assert it == g["iterations"] == math.ceil(math.log2((g["hi"] - g["lo"]) / g["tau"]))
    assert abs(lam - g["lambda_k"]) < g["tau"] / 2
    # Alg. 1' stops once the bracket holds <= m_max eigenvalues and keeps k inside it
    (lo, hi, nl, nh), it2, _ = bisect_alg1p(lambda s: oracle.nu_dense(A, B, s).n_neg, 32, 0.5, 64.5, 0, 64, m_max=4)
    assert nh - nl <= 4 and nl < 32 <= nh and lo < 32 < hi


# ---------------------------------------------------------------- P1 / P2 dense BK
@pytest.mark.parametrize("n,zero_diag,seed", [(5, False, 0), (40, False, 1), (40, True, 2), (120, True, 3), (200, False, 4)])
def test_bk_inertia_vs_eigvalsh(n, zero_diag, seed):
    rng = np.random.default_rng(seed)
    S = _rand_sym(rng, n, zero_diag)
    r = bk_ldl(S, return_factors=True)
    w = np.linalg.eigvalsh(S)
    assert (r.n_neg, r.n_zero, r.n_pos) == (int(np.sum(w < 0)), 0, int(np.sum(w > 0)))
    assert reconstruct(S, r) <= 1e-12                 # P8 on the oracle itself
    if zero_diag:
        assert r.n_2x2 > 0                            # the 2x2 path is exercised


def test_bk_vs_lapack_ldl():
    # P2: LAPACK dsytrf (scipy.linalg.ldl) is Bunch-Kaufman too; inertia of its D must agree
    rng = np.random.default_rng(7)
    for n in (10, 60, 150):
        S = _rand_sym(rng, n, zero_diag=(n == 60))
        _, D, _ = sla.ldl(S, lower=True)
        w = np.linalg.eigvalsh(D)
        r = bk_ldl(S)
        assert r.n_neg == int(np.sum(w < 0)) and r.n_pos == int(np.sum(w > 0))


def test_block_inertia_2x2_cases():
    rng = np.random.default_rng(3)
    for _ in range(500):
        d11, d21, d22 = rng.standard_normal(3) * rng.choice([1e-3, 1, 1e3], 3)
        neg, zer, pos, mn = block_inertia_2x2(d11, d21, d22)
        w = np.linalg.eigvalsh(np.array([[d11, d21], [d21, d22]]))
        assert (neg, pos) == (int(np.sum(w < 0)), int(np.sum(w > 0)))
        assert math.isclose(mn, np.min(np.abs(w)), rel_tol=1e-9)
    assert block_inertia_2x2(-1.0, 0.0, -2.0)[:3] == (2, 0, 0)
    assert block_inertia_2x2(2.0, 1.0, 3.0)[:3] == (0, 0, 2)
    assert block_inertia_2x2(-2.0, 1.0, -3.0)[:3] == (2, 0, 0)
    assert block_inertia_2x2(1.0, 1.0, 1.0)[:3] == (0, 1, 1)


def test_bk_singular_detected():
    S = np.array([[1.0, 1.0], [1.0, 1.0]])
    r = bk_ldl(S)
    assert r.singular and r.n_zero == 1
    S3 = np.zeros((3, 3))
    assert bk_ldl(S3).n_zero == 3


# ---------------------------------------------------------------- P1 pencils (dense and sparse)
@pytest.mark.parametrize("n,seed", [(50, 0), (100, 1), (200, 2)])
def test_random_pencils_nu(n, seed):
    rng = np.random.default_rng(seed)
    A, B = _rand_pencil(rng, n)
    w = oracle.eigvals_pencil(A, B)
    sig = rng.uniform(w[0] - 1, w[-1] + 1, 20)
    for s in sig:
        assert oracle.nu_dense(A, B, s).n_neg == oracle.nu_eig(A, B, s, eigvals=w)


def test_c1_dense_sparse_eig_agree():
    p = kepgen.config(1)
    A, B = p.dense("a"), p.dense("b")
    w = oracle.eigvals_pencil(A, B)
    sig = kepgen.uniform_shifts(w[0], w[-1], 32)
    so = oracle.SparseOracle(p)
    for i, s in enumerate(sig):
        ref = oracle.nu_eig(A, B, s, eigvals=w)
        assert so.inertia(s).n_neg == ref
        if i % 8 == 3:
            assert oracle.nu_dense(A, B, s).n_neg == ref


def test_sparse_oracle_delays_and_orderings():
    # u = 0.5 forces many delayed pivots; nu must not change (ordering / pivot invariance)
    p = kepgen.tb_pencil(shape=(4, 4, 5), o=3, seed=11)
    A, B = p.dense("a"), p.dense("b")
    w = oracle.eigvals_pencil(A, B)
    sig = kepgen.uniform_shifts(w[0], w[-1], 12)
    delayed = 0
    for ordering in ("nd", "rcm", "natural"):
        so = oracle.SparseOracle(p, ordering=ordering)
        for s in sig:
            for u in (0.01, 0.5):
                r = so.inertia(s, u=u)
                delayed += r.n_delayed
                assert r.n_neg == oracle.nu_eig(A, B, s, eigvals=w)
    assert delayed > 0


# ---------------------------------------------------------------- P4 closed-form twins
@pytest.mark.parametrize("shape,o,per,uA", [((4, 4, 6), 3, (False, False, False), 0.0),
                                            ((3, 4, 5), 2, (False, False, True), 0.1),
                                            ((5, 3, 4), 4, (True, False, False), 0.05)])
def test_twin_closed_form_vs_eigh(shape, o, per, uA):
    q = kepgen.twin_pencil(shape, o, periodic=per, uA=uA, uB=0.01, seed=101)
    w = oracle.twin_eigenvalues(q.meta["twin"])
    we = oracle.eigvals_pencil(q.dense("a"), q.dense("b"))
    assert np.max(np.abs(w - we)) <= 1e-12 * max(1.0, np.max(np.abs(we)))
    so = oracle.SparseOracle(q)
    for s in kepgen.uniform_shifts(w[0], w[-1], 10):
        assert so.inertia(s).n_neg == oracle.nu_twin(q.meta["twin"], s, w)


def test_twin_sparse_mid_size():
    # n = 6400, beyond comfortable dense range: O-sparse vs the closed form
    q = kepgen.twin_pencil((8, 10, 20), 4, seed=102)
    w = oracle.twin_eigenvalues(q.meta["twin"])
    so = oracle.SparseOracle(q)
    for s in kepgen.uniform_shifts(w[0], w[-1], 6):
        assert so.inertia(s).n_neg == oracle.nu_twin(q.meta["twin"], s, w)


# ---------------------------------------------------------------- P5 Sturm
def test_sturm_and_chain():
    rng = np.random.default_rng(5)
    n = 300
    d = rng.uniform(-2, 2, n)
    e = rng.uniform(-1, 1, n - 1)
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    w = np.linalg.eigvalsh(T)
    # a 1-D chain pencil (B = I) in kepgen storage, natural ordering
    colptr = np.zeros(n + 1, dtype=np.int64)
    rows, a = [], []
    for j in range(n):
        rows += [j] + ([j + 1] if j + 1 < n else [])
        a += [d[j]] + ([e[j]] if j + 1 < n else [])
        colptr[j + 1] = len(rows)
    b = np.array([1.0 if r == j else 0.0 for j in range(n) for r in ([j] + ([j + 1] if j + 1 < n else []))])
    p = kepgen.Pencil(n=n, colptr=colptr, rowidx=np.array(rows, np.int32), a=np.array(a), b=b, o=1)
    so = oracle.SparseOracle(p, ordering="natural")
    for s in rng.uniform(w[0] - 0.5, w[-1] + 0.5, 25):
        ref = int(np.sum(w < s))
        assert sturm_count(d, e, s) == ref
        assert so.inertia(s).n_neg == ref


# ---------------------------------------------------------------- P6 metamorphic
def test_metamorphic_identities():
    p = kepgen.tb_pencil(shape=(3, 4, 5), o=2, seed=21)
    A, B = p.dense("a"), p.dense("b")
    n = p.n
    w = oracle.eigvals_pencil(A, B)
    so = oracle.SparseOracle(p)
    rng = np.random.default_rng(0)
    sig = np.sort(rng.uniform(w[0], w[-1], 10))
    prev = -1
    for s in sig:
        v = oracle.nu_dense(A, B, s).n_neg
        assert v >= prev                                               # (vi) monotone
        prev = v
        tau = 0.37
        assert oracle.nu_dense(A + tau * B, B, s + tau).n_neg == v     # (iii) shift
        assert oracle.nu_dense(-A, B, -s).n_neg == n - v               # (iv) negation
        assert oracle.nu_dense(2.5 * A, 2.5 * B, s).n_neg == v         # (v) scaling
        # (i) per-atom block congruence X^T S X keeps the pattern and the inertia
        X = np.kron(np.eye(p.natoms), rng.standard_normal((2, 2)) + 2 * np.eye(2))
        assert oracle.nu_dense(X.T @ A @ X, X.T @ B @ X, s).n_neg == v
        assert so.inertia(s).n_neg == v
    rho = np.max(np.sum(np.abs(A), axis=1)) / np.min(np.linalg.eigvalsh(B))
    assert oracle.nu_dense(A, B, -rho - 1).n_neg == 0 and oracle.nu_dense(A, B, rho + 1).n_neg == n   # (vii)


# ---------------------------------------------------------------- P9 symbolic brute force
def test_brute_symbolic_closed_forms():
    n = 12
    # tridiagonal, natural order: no fill, path etree
    colptr = np.arange(0, 2 * n, 2, dtype=np.int64)
    colptr = np.append(colptr, 2 * n - 1)
    rowidx = np.array([x for j in range(n) for x in ([j, j + 1] if j + 1 < n else [j])])
    counts, parent = brute_symbolic(n, colptr, rowidx, np.arange(n))
    assert np.sum(counts) == 2 * n - 1 and list(parent[:-1]) == list(range(1, n))
    # arrowhead (dense first column): natural order fills everything, arrow last gives O(n)
    rows = [np.arange(n)] + [np.array([j]) for j in range(1, n)]
    colptr = np.cumsum([0] + [len(r) for r in rows]).astype(np.int64)
    rowidx = np.concatenate(rows)
    c_nat, _ = brute_symbolic(n, colptr, rowidx, np.arange(n))
    pos = np.array([n - 1] + list(range(n - 1)))
    c_arr, _ = brute_symbolic(n, colptr, rowidx, pos)
    assert np.sum(c_nat) == n * (n + 1) // 2 and np.sum(c_arr) == 2 * n - 1
    # diagonal: every column a root, nzf = n
    c_d, par_d = brute_symbolic(n, np.arange(n + 1, dtype=np.int64), np.arange(n), np.arange(n))
    assert np.sum(c_d) == n and np.all(par_d == -1)


# ---------------------------------------------------------------- blocked O-sparse panel
@pytest.mark.parametrize("f,q,zero_diag,u,seed", [(60, 40, True, 0.01, 0), (60, 40, True, 0.5, 1),
                                                  (90, 90, True, 0.01, 2), (80, 30, False, 0.3, 3),
                                                  (120, 70, True, 0.45, 4)])
def test_blocked_panel_matches_unblocked_front(f, q, zero_diag, u, seed):
    """The blocked front kernel takes the unblocked loop's decisions: same pivot order,
    delays, 2x2 count and inertia, and the same contribution block (rounding only)."""
    from oracle.sparse_mf import _partial_fs_bk, _partial_fs_bk_blocked
    rng = np.random.default_rng(seed)
    S = _rand_sym(rng, f, zero_diag)
    root = q == f
    F0 = S.copy()
    r0, o0, e0 = _partial_fs_bk(F0, q, u=u, root=root)
    for nb in (1, 2, 5, 16, 64):
        F1 = np.asfortranarray(S.copy())
        r1, o1, e1 = _partial_fs_bk_blocked(F1, q, u=u, root=root, nb=nb)
        assert e1 == e0 and np.array_equal(o1, o0)
        assert (r1.n_neg, r1.n_pos, r1.n_zero, r1.n_2x2, r1.n_delayed) == \
               (r0.n_neg, r0.n_pos, r0.n_zero, r0.n_2x2, r0.n_delayed)
        assert np.allclose(F1[e0:, e0:], F0[e0:, e0:], rtol=0, atol=1e-11 * np.max(np.abs(S)))
    if root:    # a root runs plain BK: its inertia is the matrix's (eigvalsh)
        w = np.linalg.eigvalsh(S)
        assert (r0.n_neg, r0.n_pos) == (int(np.sum(w < 0)), int(np.sum(w > 0)))


def test_blocked_sparse_oracle_vs_eigh_and_unblocked():
    # u = 0.5 forces delays; the blocked oracle must agree with eigh (P1) and the unblocked loop
    p = kepgen.tb_pencil(shape=(5, 5, 6), o=4, seed=12)
    A, B = p.dense("a"), p.dense("b")
    w = oracle.eigvals_pencil(A, B)
    so = oracle.SparseOracle(p)
    delayed = 0
    for s in kepgen.uniform_shifts(w[0], w[-1], 8):
        for u in (0.01, 0.5):
            r0 = so.inertia(s, u=u)
            r1 = so.inertia(s, u=u, nb=8)
            assert r1.n_neg == oracle.nu_eig(A, B, s, eigvals=w)
            assert (r1.n_neg, r1.n_delayed, r1.n_2x2) == (r0.n_neg, r0.n_delayed, r0.n_2x2)
            delayed += r1.n_delayed
    assert delayed > 0


def test_blocked_sparse_oracle_twin_mid_size():
    # n = 6400 with the cutoff-2.2-like pattern (c5 geometry in miniature): blocked O-sparse vs closed form
    q = kepgen.twin_pencil((8, 10, 20), 4, uA=0.08, uB=0.01, seed=106)
    w = oracle.twin_eigenvalues(q.meta["twin"])
    so = oracle.SparseOracle(q)
    for s in kepgen.uniform_shifts(w[0], w[-1], 5):
        assert so.inertia(s, nb=32).n_neg == oracle.nu_twin(q.meta["twin"], s, w)


# ---------------------------------------------------------------- f4: Brent's method on nu
def test_brent_nu_brackets_kth():
    from oracle.bisection import bisect_alg1p, brent_nu
    g = json.load(open(GOLD))["bisection"][0]                    # SPEC diag(1..64), B = I
    A = np.diag(np.arange(1, g["n"] + 1, dtype=float))
    B = np.eye(g["n"])
    nu = lambda s: oracle.nu_dense(A, B, s).n_neg
    for k in (1, 17, 32, 64):
        for m_max in (1, 4, 20):
            (lo, hi, nl, nh), it, tr = brent_nu(nu, k, 0.5, 64.5, 0, 64, m_max=m_max)
            assert nl < k <= nh and nh - nl <= m_max and lo <= k < hi      # lambda_k in [lo, hi)
            assert nl == nu(lo) and nh == nu(hi)
    # a clustered random pencil against eigh (P1): the bracket holds lambda_k, <= m_max eigenvalues
    rng = np.random.default_rng(9)
    Aa, Bb = _rand_pencil(rng, 120)
    w = oracle.eigvals_pencil(Aa, Bb)
    nu2 = lambda s: oracle.nu_eig(Aa, Bb, s, eigvals=w)
    for k in (5, 60, 118):
        (lo, hi, nl, nh), it, _ = brent_nu(nu2, k, w[0] - 1, w[-1] + 1, 0, 120, m_max=3)
        assert lo <= w[k - 1] < hi and nh - nl <= 3 and nl == int(np.sum(w < lo))
        _, it_b, _ = bisect_alg1p(nu2, k, w[0] - 1, w[-1] + 1, 0, 120, m_max=3)
        assert it <= 3 * it_b + 3
