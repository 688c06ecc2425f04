"""Write tests/golden/oracle_flops.json: the CPU oracle's own algorithmic flop count per
shift (O-sparse fronts from its geometric ND, sum over fronts of sum_{m=c}^{f-1} (m^2 + 2m))
for the full-size configs and for the bounded samples bench.py times.  bench.py scales
the oracle's measured sample time to a full-size shift by the ratio of these counts
(DESIGN.md §6).  Calls only oracle/ and the seeded generator kepgen.

    python scripts/oracle_flops.py [--configs 4]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import kepgen  # noqa: E402
from oracle.sparse_mf import SparseOracle  # noqa: E402

SAMPLES = {4: [(10, 10, 100), (10, 10, 150)]}


def oracle_flops(p):
    piv, fs = SparseOracle(p).front_sizes()
    tot = 0.0
    for pp, ff in zip(piv, fs):
        m = np.arange(ff - pp, ff, dtype=np.float64)
        tot += float(np.sum(m * m + 2 * m))
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[4])
    a = ap.parse_args()
    path = os.path.join(ROOT, "tests", "golden", "oracle_flops.json")
    doc = json.load(open(path)) if os.path.exists(path) else {"_source": "scripts/oracle_flops.py (oracle/ only)"}
    for cfg in a.configs:
        ent = {"full": oracle_flops(kepgen.config(cfg))}
        for shp in SAMPLES.get(cfg, []):
            ent["x".join(map(str, shp))] = oracle_flops(kepgen.config(cfg, shape=shp))
        doc[f"c{cfg}"] = ent
        print(cfg, ent, flush=True)
    json.dump(doc, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
