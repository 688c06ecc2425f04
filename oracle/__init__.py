"""oracle — plain, slow, obviously-correct CPU reference for nu_sigma(A, B).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` leg / ``--impl reference`` arm may import or
run anything in this package.  The product path (``paper_1710_05134_b200``)
never imports it and shares no code with it; the only shared module is the
seeded input generator ``kepgen`` (which holds none of the method's
arithmetic).

What it computes (§1; §2.1; Alg. 1 lines 3-4,
PAPER.md:103-104; Alg. 1' PAPER.md:419-420):

    nu_sigma(A, B) = #{ i : lambda_i < sigma },  A x = lambda B x,

the number of eigenvalues of the symmetric-definite pencil strictly below
sigma, which by Sylvester's law of inertia equals the number of negative
eigenvalues of the block-diagonal D of any LDL^T factorisation of
P(A - sigma B)P^T ("Due to Sylvester's law of inertia,
nu_0(D, I) equals nu_sigma(A, B)").

Modules
-------
- ``eig``         the plain definition: count of generalized eigenvalues
                  (scipy/LAPACK ``eigh``) below sigma — small n.
- ``dense_bk``    textbook Bunch-Kaufman LDL^T (PAPER.md:86 cites
                  Bunch-Kaufman 1977) with the 1x1 / 2x2 inertia rules.
- ``sparse_mf``   a plain multifrontal LDL^T (inertia only) with its own
                  geometric nested-dissection ordering Q (PAPER.md:398-403,
                  §3.3) and FS-restricted threshold Bunch-Kaufman with delayed
                  pivots (reading R1) — larger n.
- ``closed_form`` closed-form spectra: separable lattice twins,
                  tridiagonal Sturm counts (P5).
- ``symbolic``    brute-force boolean elimination (nnz of L, etree) for the
                  symbolic pins.
- ``lanczos``     stage 1 (Alg. 2, generalized Lanczos Eq. 2.1) and stage 3
                  (Alg. 3, SI Lanczos Eq. 2.4 with error bounds Eq. 3.1 and
                  tests 3.3-3.5), step by step.

Pins (what each is checked against, in ``tests/test_oracle_*.py``) are listed
in DESIGN.md §"Oracle and pins".  Parity unpinned: L, D, pivot order, delayed
pivot counts (not unique; only nu and the factor residual are).
"""
from .eig import nu_eig, eigvals_pencil
from .dense_bk import ALPHA, bk_ldl, nu_dense, block_inertia_2x2, Inertia, reconstruct
from .closed_form import twin_eigenvalues, nu_twin, sturm_count
from .sparse_mf import nu_sparse, SparseOracle
from .lanczos import lanczos_decomposition, initial_interval_alg2, si_lanczos_alg3, tridiag_eig

__all__ = [
    "nu_eig", "eigvals_pencil", "ALPHA", "bk_ldl", "nu_dense", "block_inertia_2x2",
    "Inertia", "reconstruct", "twin_eigenvalues", "nu_twin", "sturm_count",
    "nu_sparse", "SparseOracle", "lanczos_decomposition", "initial_interval_alg2", "si_lanczos_alg3",
    "tridiag_eig",
]
