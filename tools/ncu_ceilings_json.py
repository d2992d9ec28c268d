"""Per-kernel utilisation of the candidate ceilings from one `ncu --set full`
report, merged into profiles/ceilings.json under a workload key (bench.py
attaches the dominant kernel's entry to its roofline line).
Usage: ncu_ceilings_json.py REP WORKLOAD [OUT]"""
import csv, io, json, os, subprocess, sys

M = {
    "lsu_shared_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "shared_atom_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum.pct_of_peak_sustained_elapsed",
    "l1_lsu_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1_writeback_pct": "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed",
    "fp64_pipe_pct": "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "ipc": "sm__inst_executed.avg.per_cycle_active",
}
NAMES = {"k_motion_field": "motion_field", "k_traj_records": "traj_records",
         "k_fwd_cells": "fwd_owner", "k_bwd_event": "bwd_event", "k_bwd_cells": "bwd_owner"}
rep, wl = sys.argv[1], sys.argv[2]
out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(__file__), "..", "profiles",
                                                            "ceilings.json")
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[0]
res = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
    key = NAMES.get(name)
    if key is None or key in res:
        continue
    e = {}
    for k, m in M.items():
        try:
            e[k] = round(float(r[hdr.index(m)]), 2)
        except (ValueError, IndexError):
            pass
    pct = {k: v for k, v in e.items() if k.endswith("_pct") and k != "issue_active_pct"}
    e["binding"] = max(pct, key=pct.get) if pct else None
    res[key] = e
try:
    with open(out) as f:
        allc = json.load(f)
except Exception:
    allc = {"_source": "tools/ncu_ceilings_json.py over one `ncu --set full --clock-control none` "
                       "capture per workload (first launch of each stage kernel)"}
allc[wl] = res
with open(out, "w") as f:
    json.dump(allc, f, indent=1)
print(json.dumps(res, indent=1))
