"""c3 factor + solves + fused SpMV, for ncu captures of k_fwd / k_bwd / k_spmv2 (dev)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import kepgen
from paper_1710_05134_b200 import Kep
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from prof_levels import cached  # noqa: E402

p, lo, hi = cached(3)
k = Kep.from_pencil(p, max_batch=1)
k.set_values(p.a, p.b)
fac = k.factor(lo + 0.4 * (hi - lo))
b = np.random.default_rng(0).standard_normal((p.n, 3))
import torch
torch.cuda.synchronize()
t = time.time()
x = fac.solve(b)
print("3 solves", time.time() - t, "s", flush=True)
lam, xv, rep = k.kth_eigenpair(int(0.25 * p.n), shifts_per_round=16, max_si=60)
print("kth", rep["status"], rep["stage3_iters"], rep["seconds"])
