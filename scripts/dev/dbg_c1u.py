"""c1, u = 0.5: nu vs eigh for nrelax / env combinations (debug)."""
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
nr = int(sys.argv[1]); u = float(sys.argv[2])
k = Kep.from_pencil(p, pivot_u=u, nrelax=nr)
k.set_values(p.a, p.b)
nus, st = k.inertia_many(sig)
bad = np.nonzero(nus != ref)[0]
print(f"nrelax={nr} u={u} env={[(x, os.environ[x]) for x in os.environ if x.startswith('KEP_')]} bad={len(bad)} first={bad[:5]}")
