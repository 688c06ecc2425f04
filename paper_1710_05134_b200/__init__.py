"""paper_1710_05134_b200 — B200-native nu_sigma(A, B) (arXiv 1710.05134 hot path).

The product is the C-ABI shared library ``lib/libkep.so`` (declared in
``include/kep.h``): hand-written sm_100a CUDA for the numeric sparse
LDL^T-with-inertia of A - sigma B, plus the host symbolic analysis.
``kep`` is the ctypes binding; ``multisection`` is the host driver of stage 2
(Alg. 1') generalised to P shifts per round over GPUs.
"""
from .kep import Factor, Kep, KepError, lib, version, LIB_PATH

__all__ = ["Factor", "Kep", "KepError", "lib", "version", "LIB_PATH"]
