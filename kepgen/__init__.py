"""kepgen — seeded synthetic pencils (A, B) for the nu_sigma(A,B) hot path.

This module is the ONE piece of code shared by the oracle (``oracle/``) and the
CUDA path (``paper_1710_05134_b200``).  It holds no arithmetic of the method
(no LDL^T, no pivoting, no inertia): it only draws random matrices with the
shapes, value distributions and sparsity structure of the paper's workloads
(Table 1, PAPER.md:781-794 Appendix: atoms, orbitals, blocks
decaying with distance, B SPD with unit-ish diagonal) as fixed by
BASELINE.json ``configs`` and SURVEY.md §8(c) reading 10.

Public API
----------
- :func:`tb_pencil`     tight-binding pencil on a jittered lattice (configs c1-c5)
- :func:`config`        the BASELINE.json configurations by index 1..5
- :func:`twin_pencil`   separable lattice "twin" pencils whose spectrum has a
                        closed form (the formula lives in ``oracle/closed_form.py``)
- :class:`Pencil`       container (lower CSC of the union pattern, values of A, B)
"""
from .pencil import Pencil, lower_csc_from_coo, full_from_lower
from .tb import tb_pencil, config, CONFIGS
from .twin import twin_pencil
from .shifts import spectral_bounds, uniform_shifts

__all__ = [
    "Pencil", "lower_csc_from_coo", "full_from_lower",
    "tb_pencil", "config", "CONFIGS", "twin_pencil",
    "spectral_bounds", "uniform_shifts",
]
