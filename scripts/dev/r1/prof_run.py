"""Small fixed workload for ncu captures: c4 recipe on a 10x10x200 wire, 8 shifts, one batch."""
import sys
sys.path.insert(0, ".")
import numpy as np
import kepgen
from paper_1710_05134_b200 import Kep

shape = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "10x10x200").split("x"))
p = kepgen.tb_pencil(shape=shape, o=4, periodic=(False, False, True), seed=4)
lo, hi = -6.5, 6.5
sig = kepgen.uniform_shifts(lo, hi, 8)
k = Kep.from_pencil(p, max_batch=8)
k.set_values(p.a, p.b)
nus, st = k.inertia_many(sig)
nus, st = k.inertia_many(sig)
print("nus", nus.tolist(), "st", st.tolist())
