"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the
bench's stage kernels from `ncu --set full` reports -> profiles/traffic.json,
which bench.py reads for the roofline object's `traffic` field.
Usage: ncu_traffic.py WORKLOAD=REPORT [WORKLOAD=REPORT ...]"""
import csv
import io
import json
import os
import subprocess
import sys

STAGE = {"k_motion_field": "motion_field", "k_traj_records": "traj_records",
         "k_fwd_cells": "fwd_owner", "k_bwd_event": "bwd_event", "k_bwd_cells": "bwd_owner"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                    "traffic.json")
try:  # merge: workloads not given keep their earlier capture
    with open(path) as f:
        out = json.load(f)
except Exception:
    out = {}
out["_source"] = ("tools/ncu_traffic.py over one `ncu --set full --clock-control none` capture "
                  "per workload (dram__bytes_read.sum + dram__bytes_write.sum per launch)")
for arg in sys.argv[1:]:
    wl, rep = arg.split("=", 1)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].split("<")[0].replace("void ", "").strip()
        if name not in STAGE:
            continue
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(m)
            tot += float(r[i]) * SCALE.get(units[i], 1)
        res.setdefault(STAGE[name], int(tot))
    out[wl] = res
with open(path, "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
