"""Per-level kernel-class times (KEP_PROFILE_LEVELS) for one config: dev profiling only.

    python scripts/dev/prof_levels.py [cfg] [shifts] [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["KEP_PROFILE_LEVELS"] = "1"
import numpy as np  # noqa: E402

import kepgen  # noqa: E402
from paper_1710_05134_b200 import Kep  # noqa: E402


def cached(cfg, shape=None):
    path = f"/root/.cache/kep_c{cfg}{'_' + 'x'.join(map(str, shape)) if shape else ''}.npz"
    if os.path.exists(path):
        z = np.load(path)
        return kepgen.Pencil(n=int(z["n"]), colptr=z["colptr"], rowidx=z["rowidx"], a=z["a"], b=z["b"], o=int(z["o"])), \
            float(z["lo"]), float(z["hi"])
    p = kepgen.config(cfg, shape=shape)
    lo, hi = kepgen.spectral_bounds(p)
    os.makedirs("/root/.cache", exist_ok=True)
    np.savez(path, n=p.n, colptr=p.colptr, rowidx=p.rowidx, a=p.a, b=p.b, o=p.o, lo=lo, hi=hi)
    return p, lo, hi


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    shape = tuple(int(x) for x in sys.argv[4].split("x")) if len(sys.argv) > 4 else None
    t = time.time()
    p, lo, hi = cached(cfg, shape)
    print(f"gen {time.time() - t:.1f}s n={p.n}", flush=True)
    kw = {}
    if os.environ.get("KEP_NRELAX"):
        kw["nrelax"] = int(os.environ["KEP_NRELAX"])
    if os.environ.get("KEP_RELAX_FRAC"):
        kw["relax_frac"] = float(os.environ["KEP_RELAX_FRAC"])
    k = Kep.from_pencil(p, max_batch=m, profile=True, **kw)
    a = k.analysis()
    print(kw, {x: a[x] for x in ("n_fronts", "n_levels", "max_front", "flops", "flops_exec", "arena_bytes", "batch")}, flush=True)
    k.set_values(p.a, p.b)
    sig = kepgen.uniform_shifts(lo, hi, m)
    k.inertia_many(sig)
    k.reset_profile()
    import torch  # noqa: E402
    torch.cuda.synchronize()
    t = time.time()
    for _ in range(reps):
        nus, st, infos = k.inertia_many(sig, with_info=True)
    dt = time.time() - t
    pr = k.profile()
    print(f"{m * reps / dt:.3f} shifts/s wall ({dt / reps * 1e3:.1f} ms per {m} shifts); redo/shift "
          f"{np.mean([i.n_redo for i in infos]):.1f} delayed/shift {np.mean([i.n_delayed for i in infos]):.1f}")
    print({kk: round(v / reps, 2) for kk, v in pr["ms"].items()}, "launches", {kk: v // reps for kk, v in pr["launches"].items()})
    print("schur TF/s", pr["schur_flops"] / ((pr["ms"]["schur"] + pr["ms"]["schur_tma"]) / 1e3) / 1e12,
          "long-K (tma) TF/s", pr["schur_tma_flops"] / max(pr["ms"]["schur_tma"] / 1e3, 1e-9) / 1e12)
    k.close()


if __name__ == "__main__":
    main()
