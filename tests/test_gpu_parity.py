"""GPU parity: the CUDA path (through the C ABI) against the oracle.

nu_sigma is an integer: the bar is bit-exact equality on every shift whose
gap to the spectrum is certified (readings R4/R5).  Inputs are the
seeded kepgen pencils; expected values come only from ``oracle/``.
"""
import json
import os

import numpy as np
import pytest

import kepgen
import oracle
from paper_1710_05134_b200 import Kep
from paper_1710_05134_b200.kep import KEP_ESINGULAR, KEP_OK

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _certified(w, sig, rel=1e-6):
    scale = max(abs(w[0]), abs(w[-1]))
    gaps = np.min(np.abs(sig[:, None] - w[None, :]), axis=1) / scale
    return gaps >= rel


def _pencil_from_dense(A, B, tol=0.0):
    n = A.shape[0]
    mask = (np.abs(np.tril(A)) > tol) | (np.abs(np.tril(B)) > tol)
    mask |= np.eye(n, dtype=bool)
    cols, rows = [], []
    colptr = [0]
    for j in range(n):
        r = np.nonzero(mask[j:, j])[0] + j
        rows.append(r)
        colptr.append(colptr[-1] + len(r))
    rowidx = np.concatenate(rows).astype(np.int32)
    colidx = np.repeat(np.arange(n), np.diff(colptr))
    return kepgen.Pencil(n=n, colptr=np.array(colptr, np.int64), rowidx=rowidx,
                         a=A[rowidx, colidx].copy(), b=B[rowidx, colidx].copy(), o=1)


def test_spec_examples_on_gpu():
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    for case in g["nu"]:
        A = np.diag(np.array(case["A_diag"], float))
        B = np.diag(np.array(case["B_diag"], float))
        p = _pencil_from_dense(A, B)
        k = Kep.from_pencil(p)
        k.set_values(p.a, p.b)
        st, nu, _ = k.inertia(case["sigma"])
        assert st == KEP_OK and nu == case["nu"], case["cite"]
    for case in g["inertia"]:
        S = np.array(case["S"], float)
        p = _pencil_from_dense(S, np.zeros_like(S), tol=-1)     # dense pattern
        k = Kep.from_pencil(p)
        k.set_values(p.a, p.b)
        st, nu, info = k.inertia(0.0)
        assert st == KEP_OK
        assert (info.n_neg, info.n_zero, info.n_pos, info.n_2x2) == (case["neg"], case["zero"], case["pos"], case["n2x2"]), case["cite"]


def test_singular_shift_reported():
    A = np.diag(np.arange(1.0, 11.0))
    p = _pencil_from_dense(A, np.eye(10))
    k = Kep.from_pencil(p)
    k.set_values(p.a, p.b)
    st, nu, info = k.inertia(4.0)       # sigma equals lambda_4: exact zero pivot
    assert st == KEP_ESINGULAR and nu is None and info.n_zero >= 1


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("u,ordering", [(0.01, "auto"), (0.5, "auto"), (0.01, "natural")])
def test_c1_all_shifts(u, ordering, variant):
    p = kepgen.config(1)
    A, B = p.dense("a"), p.dense("b")
    w = oracle.eigvals_pencil(A, B)
    sig = kepgen.uniform_shifts(w[0], w[-1], 32)
    assert np.all(_certified(w, sig))
    ref = oracle.nu_eig(A, B, sig, eigvals=w)
    k = Kep.from_pencil(p, pivot_u=u, ordering=ordering, kernel_variant=variant)
    k.set_values(p.a, p.b)
    nus, per, infos = k.inertia_many(sig, with_info=True)
    assert np.all(per == KEP_OK)
    assert np.array_equal(nus, ref)
    for s, i in zip(sig, infos):
        assert i.n_neg + i.n_zero + i.n_pos == p.n
    if u == 0.5:
        assert sum(i.n_delayed for i in infos) > 0       # delayed pivots exercised
    # single-shift entry point agrees with the batched one
    st, nu, _ = k.inertia(sig[7])
    assert st == KEP_OK and nu == ref[7]


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("n,seed", [(40, 0), (90, 1)])
def test_random_dense_pencils(n, seed, variant):
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, n))
    A = M + M.T
    np.fill_diagonal(A, 0.0)                 # forces 2x2 pivots
    R = rng.standard_normal((n, n))
    B = R.T @ R + n * np.eye(n)
    p = _pencil_from_dense(A, B, tol=-1)
    w = oracle.eigvals_pencil(A, B)
    sig = rng.uniform(w[0] - 0.1, w[-1] + 0.1, 24)
    sig = sig[_certified(w, sig)]
    k = Kep.from_pencil(p, kernel_variant=variant)
    k.set_values(p.a, p.b)
    nus, per, infos = k.inertia_many(sig, with_info=True)
    assert np.all(per == KEP_OK)
    assert np.array_equal(nus, oracle.nu_eig(A, B, sig, eigvals=w))
    assert sum(i.n_2x2 for i in infos) > 0


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("shape,o,per,uA,u", [((6, 6, 8), 4, (False, False, False), 0.0, 0.01),
                                              ((5, 4, 12), 2, (False, False, True), 0.08, 0.01),
                                              ((6, 6, 8), 4, (False, False, False), 0.0, 0.5)])
def test_twins_closed_form(shape, o, per, uA, u, variant):
    q = kepgen.twin_pencil(shape, o, periodic=per, uA=uA, uB=0.01, seed=103)
    w = oracle.twin_eigenvalues(q.meta["twin"])
    sig = kepgen.uniform_shifts(w[0], w[-1], 24)
    sig = sig[_certified(w, sig)]
    k = Kep.from_pencil(q, pivot_u=u, kernel_variant=variant)
    k.set_values(q.a, q.b)
    nus, st = k.inertia_many(sig)
    assert np.all(st == KEP_OK)
    assert np.array_equal(nus, oracle.nu_twin(q.meta["twin"], sig, w))


def test_metamorphic_on_gpu():
    p = kepgen.tb_pencil(shape=(4, 4, 6), o=3, seed=31)
    A, B = p.dense("a"), p.dense("b")
    w = oracle.eigvals_pencil(A, B)
    sig = kepgen.uniform_shifts(w[0], w[-1], 12)
    sig = sig[_certified(w, sig)]
    k = Kep.from_pencil(p)
    k.set_values(p.a, p.b)
    base, _ = k.inertia_many(sig)
    assert np.all(np.diff(base) >= 0)                              # monotone in sigma
    tau = 0.41
    k.set_values(p.a + tau * p.b, p.b)
    shifted, _ = k.inertia_many(sig + tau)
    k.set_values(-p.a, p.b)
    neg, _ = k.inertia_many(-sig)
    k.set_values(3.0 * p.a, 3.0 * p.b)
    scl, _ = k.inertia_many(sig)
    assert np.array_equal(shifted, base) and np.array_equal(neg, p.n - base) and np.array_equal(scl, base)


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_full_size_goldens(cfg):
    """BASELINE full sizes: nu at the certified shifts stored by scripts/make_goldens.py (oracle only)."""
    path = os.path.join(GOLD, f"c{cfg}_nu.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    g = json.load(open(path))
    p = kepgen.config(cfg)
    assert p.n == g["n"] and p.nnz == g["nnz_lower"]
    sig = np.array([x["sigma"] for x in g["shifts"]])
    k = Kep.from_pencil(p)
    k.set_values(p.a, p.b)
    nus, st = k.inertia_many(sig)
    assert np.all(st == KEP_OK)
    checked = 0
    for x, v in zip(g["shifts"], nus):
        if x["certified"]:
            assert v == x["nu"], (x["sigma"], v, x["nu"])
            checked += 1
    assert checked >= len(sig) // 2


def test_twin_c4_geometry_full_size():
    """n = 1.5M closed-form twin with the c4 geometry (10x10x3750, periodic z, o = 4)."""
    q = kepgen.twin_pencil((10, 10, 3750), 4, periodic=(False, False, True), seed=104)
    w = oracle.twin_eigenvalues(q.meta["twin"])
    sig = kepgen.uniform_shifts(w[0], w[-1], 40)
    sig = sig[_certified(w, sig)]
    assert sig.shape[0] >= 24
    k = Kep.from_pencil(q)
    k.set_values(q.a, q.b)
    nus, st = k.inertia_many(sig)
    assert np.all(st == KEP_OK)
    assert np.array_equal(nus, oracle.nu_twin(q.meta["twin"], sig, w))


def test_twin_c5_geometry_full_size():
    """n = 500k closed-form twin with the c5 geometry (50^3, o = 4) and the cutoff-2.2-like
    27+6-point pattern: root FS block ~20k columns, i.e. the global-scratch pivot-block path
    of k_fsp (FS blocks too large for shared memory) and the multi-CTA trailing updates."""
    q = kepgen.twin_pencil((50, 50, 50), 4, uA=0.08, uB=0.01, seed=105)
    w = oracle.twin_eigenvalues(q.meta["twin"])
    sig = kepgen.uniform_shifts(w[0], w[-1], 6)
    sig = sig[_certified(w, sig)][:4]
    assert sig.shape[0] >= 2
    k = Kep.from_pencil(q, max_batch=2)
    assert k.analysis()["max_front"] > 4000
    k.set_values(q.a, q.b)
    nus, st = k.inertia_many(sig)
    assert np.all(st == KEP_OK)
    assert np.array_equal(nus, oracle.nu_twin(q.meta["twin"], sig, w))


@pytest.mark.parametrize("u", [0.01, 0.5])
def test_big_front_path_c1_c2(monkeypatch, u):
    """kernels_big.cu (multi-CTA panel of the top-level fronts) routed onto the c1 / c2 top levels
    (KEP_BIG_Q lowers its FS threshold): nu equals LAPACK eigh at every certified shift (c1, with
    u = 0.5 many delays) and the stored factor reconstructs A - sigma B (front-local residual bound)."""
    monkeypatch.setenv("KEP_BIG_Q", "48")
    p = kepgen.config(1)
    A, B = p.dense("a"), p.dense("b")
    w = oracle.eigvals_pencil(A, B)
    sig = kepgen.uniform_shifts(w[0], w[-1], 32)
    sig = sig[_certified(w, sig)]
    k = Kep.from_pencil(p, pivot_u=u)
    k.set_values(p.a, p.b)
    nus, st = k.inertia_many(sig)
    assert np.all(st == KEP_OK)
    assert np.array_equal(nus, oracle.nu_eig(A, B, sig, eigvals=w))
    for s in sig[::8]:
        bound, _ = k.factor_residual(s)
        assert bound <= 1e-10 * np.linalg.norm(A - s * B)
    g = json.load(open(os.path.join(GOLD, "c2_nu.json")))
    p2 = kepgen.config(2)
    k2 = Kep.from_pencil(p2, pivot_u=u)
    k2.set_values(p2.a, p2.b)
    s2 = np.array([x["sigma"] for x in g["shifts"]])
    nus2, st2 = k2.inertia_many(s2)
    assert np.all(st2 == KEP_OK)
    for x, v in zip(g["shifts"], nus2):
        if x["certified"]:
            assert v == x["nu"]
