"""DRAM traffic per launch of one kernel from an ncu report (all captured launches).

    python scripts/ncu_traffic.py gpurun_out/x.ncu-rep k_schur > profiles/r1_schur_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

rep, name = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3,
         "msecond": 1e-3, "nsecond": 1e-9}


def val(r, key):
    i = hdr.index(key)
    return float(r[i].replace(",", "")) * scale.get(units[i], 1.0)


launches = []
for r in rows[2:]:
    if name not in r[hdr.index("Kernel Name")]:
        continue
    launches.append(dict(read=val(r, "dram__bytes_read.sum"), write=val(r, "dram__bytes_write.sum"),
                         seconds=val(r, "gpu__time_duration.sum")))
tot = sum(x["read"] + x["write"] for x in launches)
print(json.dumps({"kernel": name, "launches": len(launches), "dram_bytes_per_launch": tot / max(len(launches), 1),
                  "dram_bytes_total": tot, "seconds_total": sum(x["seconds"] for x in launches),
                  "per_launch": launches, "source": rep}, indent=1))
