"""Host-side logic of libkep.so that runs without a GPU (CPU suite).

- kep_tridiag_eigen: the Lanczos stages' tridiagonal eigensolver (Eq. (2.2),
  PAPER.md:129-134; Eq. (2.5)) against LAPACK
  (scipy.linalg.eigh_tridiagonal) and the defining identities T Z = Z diag(w),
  Z^T Z = I, including Wilkinson's W21+ (close pairs), split matrices (zero
  off-diagonals), constant diagonals and orders 1, 2.
"""
import numpy as np
import pytest
import scipy.linalg as sla

from paper_1710_05134_b200.kep import tridiag_eigen


def _cases():
    rng = np.random.default_rng(0)
    yield rng.standard_normal(50), rng.standard_normal(49)
    yield np.abs(np.arange(-10, 11)).astype(float), np.ones(20)          # W21+: pairs agree to ~1e-14
    d, e = rng.standard_normal(40), rng.standard_normal(39)
    e[[5, 17, 30]] = 0.0                                                 # split into blocks
    yield d, e
    yield np.full(30, 2.0), np.full(29, -1.0)                            # 1-D Laplacian: closed form
    yield np.array([3.0]), np.zeros(0)
    yield np.array([1.0, -1.0]), np.array([1e-300])
    yield rng.uniform(-1, 1, 200) * 1e3, rng.uniform(-1, 1, 199) * 1e-3  # nearly diagonal, wide range
    yield rng.standard_normal(300), np.abs(rng.standard_normal(299))     # Lanczos-sized


@pytest.mark.parametrize("case", list(range(8)))
def test_tridiag_eigen_vs_lapack(case):
    d, e = list(_cases())[case]
    w, Z = tridiag_eigen(d, e)
    n = d.shape[0]
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    ref = sla.eigh_tridiagonal(d, e, eigvals_only=True) if n > 1 else d.copy()
    scale = max(np.max(np.abs(T)), 1e-300)
    assert np.all(np.diff(w) >= 0)
    assert np.max(np.abs(w - ref)) <= 1e-13 * scale * max(1, np.sqrt(n))
    assert np.max(np.abs(T @ Z - Z * w)) <= 1e-13 * scale * max(1, np.sqrt(n))
    assert np.max(np.abs(Z.T @ Z - np.eye(n))) <= 1e-13 * max(1, np.sqrt(n))
    if case == 3:                                                        # 2 - 2 cos(pi j / (n + 1))
        j = np.arange(1, n + 1)
        assert np.allclose(w, 2 - 2 * np.cos(np.pi * j / (n + 1)), atol=1e-14, rtol=0)


def test_bench_config_identical_in_both_arms():
    """bench.py prints the same `config` object in the GPU arm and the reference arm (the driver
    compares them), and it names the BASELINE c4 workload."""
    import bench
    a = bench.workload_config(4, None, 1, 16)
    b = bench.workload_config(4, None, 1, 16)
    assert a == b and a["workload"] == "c4" and a["n"] == 1_500_000 and a["shifts_per_step"] == 16
    assert bench.workload_config(4, None, 8, 16)["shifts_per_step"] == 128       # BASELINE: 16 per GPU at 8


def test_oracle_flops_golden_consistent():
    """The CPU-baseline scale factors come from the oracle's own flop counts (scripts/oracle_flops.py)."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_flops.json")))["c4"]
    assert g["full"] > g["10x10x150"] > g["10x10x100"] > 0
    # the wire is uniform along z: the per-length cost of the two samples agrees within 15 %
    assert abs(g["10x10x150"] / 150 - g["10x10x100"] / 100) < 0.15 * g["10x10x100"] / 100
