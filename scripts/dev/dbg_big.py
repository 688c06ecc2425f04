import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["KEP_DEBUG_RESID"] = "1"
os.environ["KEP_BIG_Q"] = sys.argv[1] if len(sys.argv) > 1 else "48"
import numpy as np, kepgen, oracle
from paper_1710_05134_b200 import Kep
p = kepgen.config(1)
A, B = p.dense("a"), p.dense("b")
w = oracle.eigvals_pencil(A, B)
k = Kep.from_pencil(p)
k.set_values(p.a, p.b)
sigs = kepgen.uniform_shifts(w[0], w[-1], 32)
os.environ["KEP_DEBUG_DUMP"] = "20"
for i in (8,):
    print(i, k.factor_residual(sigs[i]), np.linalg.norm(A - sigs[i] * B), flush=True)
nus, st = k.inertia_many(sigs)
print("after batch")
for i in (0, 5):
    print(i, k.factor_residual(sigs[i]), np.linalg.norm(A - sigs[i] * B), flush=True)
first, parent, order = k.fronts()
print("fronts", len(parent), "piv", np.diff(first)[-8:], "order", order[-8:])
