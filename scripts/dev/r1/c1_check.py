"""c1 (BASELINE configs[0]) nu at 32 shifts against LAPACK eigh, for sanitizer runs:
    python scripts/c1_check.py <variant> <u>"""
import sys
sys.path.insert(0, ".")
import numpy as np
import kepgen
import oracle
from paper_1710_05134_b200 import Kep

variant = int(sys.argv[1]) if len(sys.argv) > 1 else 0
u = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
p = kepgen.config(1)
A, B = p.dense("a"), p.dense("b")
w = oracle.eigvals_pencil(A, B)
sig = kepgen.uniform_shifts(w[0], w[-1], 32)
ref = oracle.nu_eig(A, B, sig, eigvals=w)
k = Kep.from_pencil(p, pivot_u=u, kernel_variant=variant)
k.set_values(p.a, p.b)
for rep in range(2):
    nus, per, infos = k.inertia_many(sig, with_info=True)
    bad = np.nonzero(nus != ref)[0]
    print("variant", variant, "u", u, "rep", rep, "mismatch", bad.tolist(), "delays", sum(i.n_delayed for i in infos), "redo", sum(i.n_redo for i in infos))
