"""c1, u = 0.5, nrelax 48, KEP_BIG_Q: per-shift nu vs eigh, front / level structure (debug)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import kepgen, oracle
from paper_1710_05134_b200 import Kep
p = kepgen.config(1)
A, B = p.dense("a"), p.dense("b")
w = oracle.eigvals_pencil(A, B)
sig = kepgen.uniform_shifts(w[0], w[-1], 32)
ref = oracle.nu_eig(A, B, sig, eigvals=w)
nr = int(sys.argv[1]); u = float(sys.argv[2]); mb = int(sys.argv[3]) if len(sys.argv) > 3 else 16
k = Kep.from_pencil(p, pivot_u=u, nrelax=nr, max_batch=mb)
first, parent, order = k.fronts()
pp = np.diff(first)
lev = np.zeros(len(parent), int)
for s in range(len(parent)):
    if parent[s] >= 0: lev[parent[s]] = max(lev[parent[s]], lev[s] + 1)
for L in range(lev.max() + 1):
    m = np.nonzero(lev == L)[0]
    print("L", L, [(int(s), int(pp[s]), int(order[s])) for s in m][:8])
k.set_values(p.a, p.b)
nus, st, infos = k.inertia_many(sig, with_info=True)
print("diff", (nus - ref).tolist())
print("delayed", [i.n_delayed for i in infos][:8])
