"""Write tests/golden/c{2,3,4,5}_nu.json: oracle nu at fixed shifts of the full-size
configs, for the GPU parity tests at BASELINE sizes.

Calls only ``oracle/`` (O-sparse multifrontal) and the seeded generator
``kepgen``.  Each shift is certified by the oracle itself: nu(sigma - d) ==
nu(sigma) == nu(sigma + d), i.e. no eigenvalue within d of sigma, with
d = 1e-3 (hi - lo) / n (a thousandth of the mean eigenvalue spacing, still many
orders above the backward error of the factorisation; R5).
``--reuse FILE`` takes nu(sigma) from an earlier run at the same shifts.

    python scripts/make_goldens.py 2 [4] [--shifts 8] [--procs 8] [--reuse old.json]
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
_NB = 0


def _init(cfg, nb, threads):
    global _P, _SO, _NB
    os.environ["OPENBLAS_NUM_THREADS"] = str(threads)
    from threadpoolctl import threadpool_limits
    threadpool_limits(threads)
    import kepgen
    from oracle.sparse_mf import SparseOracle
    _P = kepgen.config(cfg)
    _SO = SparseOracle(_P)
    _NB = nb


def _nu(sigma):
    t = time.time()
    r = _SO.inertia(sigma, nb=_NB)
    return sigma, int(r.n_neg), int(r.n_delayed), bool(r.singular), time.time() - t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", type=int, nargs="+")
    ap.add_argument("--shifts", type=int, default=8)
    ap.add_argument("--procs", type=int, default=8)
    ap.add_argument("--reuse", default=None)
    ap.add_argument("--threads", type=int, default=1, help="BLAS threads per worker process")
    ap.add_argument("--nb", type=int, default=None,
                    help="O-sparse FS panel width (0 = unblocked loop); default 64 for c3 and c5, else 0")
    a = ap.parse_args()
    import numpy as np
    import kepgen
    for cfg in a.configs:
        p = kepgen.config(cfg)
        lo, hi = kepgen.spectral_bounds(p)
        sig = kepgen.uniform_shifts(lo, hi, a.shifts)
        d = 1e-3 * (hi - lo) / p.n
        old = {}
        if a.reuse:
            for x in json.load(open(a.reuse))["shifts"]:
                old[x["sigma"]] = (x["sigma"], x["nu"], x["oracle_delayed"], False, x["oracle_seconds"])
        todo = []
        for s in sig:
            todo += [s - d] + ([] if float(s) in old else [s]) + [s + d]
        nb = a.nb if a.nb is not None else (64 if cfg in (3, 5) else 0)
        with get_context("fork").Pool(a.procs, initializer=_init, initargs=(cfg, nb, a.threads)) as pool:
            res = pool.map(_nu, todo, chunksize=1)
        out = []
        it = iter(res)
        for s in sig:
            r_m = next(it)
            r_0 = old[float(s)] if float(s) in old else next(it)
            r_p = next(it)
            (_, nm, _, sm, _), (_, n0, dl, s0, t0), (_, npl, _, sp, _) = r_m, r_0, r_p
            out.append(dict(sigma=float(s), nu=n0, certified=bool(nm == n0 == npl and not (sm or s0 or sp)),
                            oracle_delayed=dl, oracle_seconds=t0))
        doc = {"_source": f"scripts/make_goldens.py: oracle.sparse_mf (O-sparse) on kepgen.config({cfg}) "
                          f"seed {kepgen.CONFIGS[cfg]['seed']}, FS panel nb={nb}; certification nu(s-d)==nu(s)==nu(s+d), d={d:.3e}",
               "config": cfg, "n": p.n, "nnz_lower": p.nnz, "lo": lo, "hi": hi, "shifts": out}
        path = os.path.join(ROOT, "tests", "golden", f"c{cfg}_nu.json")
        json.dump(doc, open(path, "w"), indent=1)
        print(path, [(o["nu"], o["certified"]) for o in out], flush=True)


if __name__ == "__main__":
    main()
