"""Write tests/golden/c{2,4}_nu.json: oracle nu at fixed shifts of the full-size
configs, for the GPU parity tests at BASELINE sizes.

Calls only ``oracle/`` (O-sparse multifrontal) and the seeded generator
``kepgen``.  Each shift is certified by the oracle itself: nu(sigma - d) ==
nu(sigma) == nu(sigma + d) with d = 1e-6 * max(|lo|, |hi|) (R5).

    python scripts/make_goldens.py 2 [4] [--shifts 8] [--procs 8]
"""
import argparse
import json
import os
import sys
import time
from multiprocessing import get_context

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

_P = None
_SO = None


def _init(cfg):
    global _P, _SO
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    import kepgen
    from oracle.sparse_mf import SparseOracle
    _P = kepgen.config(cfg)
    _SO = SparseOracle(_P)


def _nu(sigma):
    t = time.time()
    r = _SO.inertia(sigma)
    return sigma, int(r.n_neg), int(r.n_delayed), bool(r.singular), time.time() - t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", type=int, nargs="+")
    ap.add_argument("--shifts", type=int, default=8)
    ap.add_argument("--procs", type=int, default=8)
    a = ap.parse_args()
    import numpy as np
    import kepgen
    for cfg in a.configs:
        p = kepgen.config(cfg)
        lo, hi = kepgen.spectral_bounds(p)
        sig = kepgen.uniform_shifts(lo, hi, a.shifts)
        d = 1e-6 * max(abs(lo), abs(hi))
        todo = []
        for s in sig:
            todo += [s - d, s, s + d]
        with get_context("fork").Pool(a.procs, initializer=_init, initargs=(cfg,)) as pool:
            res = pool.map(_nu, todo)
        out = []
        for i, s in enumerate(sig):
            (_, nm, _, sm, _), (_, n0, dl, s0, t0), (_, npl, _, sp, _) = res[3 * i:3 * i + 3]
            out.append(dict(sigma=float(s), nu=n0, certified=bool(nm == n0 == npl and not (sm or s0 or sp)),
                            oracle_delayed=dl, oracle_seconds=t0))
        doc = {"_source": f"scripts/make_goldens.py: oracle.sparse_mf (O-sparse) on kepgen.config({cfg}) "
                          f"seed {kepgen.CONFIGS[cfg]['seed']}; certification nu(s-d)==nu(s)==nu(s+d), d={d:.3e}",
               "config": cfg, "n": p.n, "nnz_lower": p.nnz, "lo": lo, "hi": hi, "shifts": out}
        path = os.path.join(ROOT, "tests", "golden", f"c{cfg}_nu.json")
        json.dump(doc, open(path, "w"), indent=1)
        print(path, [(o["nu"], o["certified"]) for o in out], flush=True)


if __name__ == "__main__":
    main()
