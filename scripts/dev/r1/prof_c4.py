"""One batch of 8 shifts on the c4 workload for ncu captures (development aid)."""
import sys
sys.path.insert(0, ".")
import kepgen
from paper_1710_05134_b200 import Kep

p = kepgen.config(4)
lo, hi = kepgen.spectral_bounds(p)
sig = kepgen.uniform_shifts(lo, hi, 8)
k = Kep.from_pencil(p, max_batch=8)
k.set_values(p.a, p.b)
nus, st = k.inertia_many(sig)
print("nus", nus.tolist(), "st", st.tolist())
