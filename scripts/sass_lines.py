"""Aggregate ncu SASS stall samples per CUDA source line.

    ncu -i rep --page source --csv --print-source sass > sass.csv
    python scripts/sass_lines.py sass.csv kernels_front.sm_100a.cubin <kernel-substring> [top]
"""
import csv
import re
import subprocess
import sys
from collections import defaultdict

sass_csv, cubin, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
ai, si, ni = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
base = int(rows[2][ai], 16)
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# find the function section for kname, map offsets -> line
cur_fn, line, off2line = None, None, {}
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        cur_fn = m.group(1)
        continue
    if cur_fn is None or kname not in cur_fn:
        continue
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', ln)
    if m:
        line = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and line:
        off2line[int(m.group(1), 16)] = line
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ridx = [hdr.index(h) for h in reasons]
agg = defaultdict(int)
why = defaultdict(lambda: defaultdict(int))
tot = 0
for r in rows[2:]:
    try:
        a = int(r[ai], 16)
        v = int(r[si] or 0)
    except (ValueError, IndexError):
        continue
    ln = off2line.get(a - base, "?")
    agg[ln] += v
    tot += v
    for h, i in zip(reasons, ridx):
        try:
            why[ln][h] += int(r[i] or 0)
        except ValueError:
            pass
print(f"total samples {tot}")
for k, v in sorted(agg.items(), key=lambda t: -t[1])[:top]:
    w = sorted(why[k].items(), key=lambda t: -t[1])[:3]
    print(f"{v:8d} {100.0 * v / tot:5.1f}%  {k:28s} " + ", ".join(f"{h[6:]}={c}" for h, c in w if c))
