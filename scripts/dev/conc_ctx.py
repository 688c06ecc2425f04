"""Concurrency experiment: W host threads, each with its own kep context (own stream, own arena,
max_batch B), each evaluating S shifts per step; total shifts/s vs one context (dev only).

    python scripts/dev/conc_ctx.py W B S reps
"""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from scripts.dev.prof_levels import cached
import kepgen
from paper_1710_05134_b200 import Kep

W, B, S, reps = (int(x) for x in sys.argv[1:5])
p, lo, hi = cached(4)
ks = []
for w in range(W):
    k = Kep.from_pencil(p, max_batch=B, nrelax=48)
    k.set_values(p.a, p.b)
    ks.append(k)
print("arena GB/shift", ks[0].analysis()["arena_bytes"] / 1e9, "batch", [k.analysis()["batch"] for k in ks], flush=True)
sig = kepgen.uniform_shifts(lo, hi, W * S)
def run(w):
    ks[w].inertia_many(sig[w * S:(w + 1) * S])
for w in range(W): run(w)                          # warm-up
torch.cuda.synchronize()
t = time.time()
for _ in range(reps):
    th = [threading.Thread(target=run, args=(w,)) for w in range(W)]
    for x in th: x.start()
    for x in th: x.join()
dt = (time.time() - t) / reps
print(f"W={W} B={B} S={S}: {W * S / dt:.3f} shifts/s ({dt * 1e3:.1f} ms per {W * S} shifts)", flush=True)
