"""Secondary ceilings of the stage kernels from an `ncu --set
full` report: shared-memory LSU wavefronts (all / atomics) and L1 throughput as
% of peak, bank-conflict wavefronts, fp64 pipe activity, DRAM throughput.
Usage: ncu_ceilings.py REP"""
import csv
import io
import subprocess
import sys

M = {
    "lsu_shared%": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "shared_atom%": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum.pct_of_peak_sustained_elapsed",
    "bank_confl_atom": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
    "lsu_all%": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex%": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "fp64_pipe%": "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "dram%": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
}
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
print("kernel".ljust(18) + "".join(k.rjust(16) for k in M))
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").split("::")[-1][:17]
    cells = []
    for k, m in M.items():
        try:
            cells.append(r[hdr.index(m)].rjust(16))
        except ValueError:
            cells.append("-".rjust(16))
    print(name.ljust(18) + "".join(cells))
