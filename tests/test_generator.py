"""Generator (kepgen) invariants: determinism, storage, SPD B, pattern shape."""
import numpy as np

import kepgen


def test_tb_deterministic_and_valid():
    p1 = kepgen.config(1)
    p2 = kepgen.config(1)
    p1.check()
    assert p1.n == 1000 and p1.k == 300
    assert np.array_equal(p1.rowidx, p2.rowidx) and np.array_equal(p1.a, p2.a) and np.array_equal(p1.b, p2.b)
    # B SPD with lambda_min >= 0.5 (shift rule), A symmetric by construction
    w = np.linalg.eigvalsh(p1.dense("b"))
    assert w[0] >= 0.5 - 1e-12
    # neighbour-block density of the cutoff-1.8 lattice (~27 blocks per atom row, both triangles)
    blocks_per_row = (2 * p1.nnz - p1.n) / p1.n / p1.o
    assert 15 < blocks_per_row < 30


def test_tb_periodic_small():
    p = kepgen.tb_pencil(shape=(3, 3, 8), o=2, periodic=(False, False, True), seed=3)
    p.check()
    # an atom at z=0 couples to z=7 through the periodic boundary
    A = p.to_scipy("a").tocsr()
    at0 = 0            # (0,0,0)
    at7 = 7            # (0,0,7)
    assert A[at0 * 2, at7 * 2] != 0


def test_twin_pattern_is_27_point():
    q = kepgen.twin_pencil((4, 4, 4), 2, seed=100)
    q.check()
    # interior atom (1,1,1) has 27 blocks in its full row
    A = q.to_scipy("a").tocsr()
    atom = (1 * 4 + 1) * 4 + 1
    cols = A[atom * 2].indices // 2
    assert len(np.unique(cols)) == 27
