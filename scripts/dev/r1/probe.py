"""Quick timing probe of kep_inertia_many on a few configs (development aid)."""
import sys, time, json
import numpy as np
import torch
sys.path.insert(0, ".")
import kepgen
from paper_1710_05134_b200 import Kep

def run(p, nshift, variant=0, batch=16):
    t = time.time(); lo, hi = kepgen.spectral_bounds(p); tb = time.time() - t
    sig = kepgen.uniform_shifts(lo, hi, nshift)
    t = time.time(); k = Kep.from_pencil(p, max_batch=batch, kernel_variant=variant, profile=True); ta = time.time() - t
    k.set_values(p.a, p.b)
    nus, st = k.inertia_many(sig[:2])       # warm
    torch.cuda.synchronize()
    k.reset_profile()
    t = time.time(); nus, st, infos = k.inertia_many(sig, with_info=True); dt = time.time() - t
    prof = k.profile()
    a = k.analysis()
    print(json.dumps(dict(name=p.name, n=p.n, analyze_s=ta, bounds_s=tb, shifts=nshift, s_per_shift=dt / nshift,
                          shifts_per_s=nshift / dt, gflops=a["flops"] * nshift / dt / 1e9, nus=nus.tolist()[:8],
                          st=st.tolist()[:8], sigma=sig.tolist()[:8], profile=prof, analysis=a, redo_per_shift=sum(i.n_redo for i in infos) / nshift,
                          delayed_per_shift=sum(i.n_delayed for i in infos) / nshift, n2x2_per_shift=sum(i.n_2x2 for i in infos) / nshift)), flush=True)

which = sys.argv[1:] or ["c1", "c2"]
for w in which:
    if w == "c1": run(kepgen.config(1), 32)
    if w == "c2": run(kepgen.config(2), 16)
    if w == "c4s": run(kepgen.tb_pencil(shape=(10, 10, 400), o=4, periodic=(False, False, True), seed=4), 16)
    if w == "c3": run(kepgen.config(3), 8, batch=8)
    if w == "c5": run(kepgen.config(5), 2, batch=2)
