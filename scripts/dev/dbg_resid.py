import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["KEP_DEBUG_RESID"] = "1"
os.environ["KEP_DEBUG_DUMP"] = "38"
import numpy as np, kepgen, oracle
from paper_1710_05134_b200 import Kep
p = kepgen.config(1)
A, B = p.dense("a"), p.dense("b")
w = oracle.eigvals_pencil(A, B)
k = Kep.from_pencil(p, kernel_variant=1)
k.set_values(p.a, p.b)
sig = kepgen.uniform_shifts(w[0], w[-1], 4)[1]
print(k.factor_residual(sig), flush=True)
S = A - sig * B
fac = k.factor(sig)
perm, d, ds, cp, ri, vals = fac.export()
np.savez("gpurun_out/dbg_c1.npz", perm=perm, d=d, ds=ds, cp=cp, ri=ri, vals=vals, S=S, kperm=k.perm())
