"""One line per kernel launch from an ncu report: duration, DRAM, IPC, occupancy,
instructions, top stall reasons. Usage: ncu_summary.py REP"""
import csv, io, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
units = rows[1]
SCALE = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3,
         "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "KB": 1e-3, "MB": 1.0, "GB": 1e3}


def val(r, name, default=0.0):
    try:
        i = hdr.index(name)
        return float(r[i]) * SCALE.get(units[i], 1.0)
    except (ValueError, IndexError):
        return default


def col(r, name):
    try:
        return r[hdr.index(name)]
    except (ValueError, IndexError):
        return ""


for r in rows[2:]:
    name = col(r, "Kernel Name").split("(")[0]
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                stalls.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    tot = sum(v for v, _ in stalls) or 1
    st = " ".join(f"{n}:{100 * v / tot:.0f}%" for v, n in stalls[:4])
    dur = val(r, "gpu__time_duration.sum")
    rd = val(r, "dram__bytes_read.sum")
    wr = val(r, "dram__bytes_write.sum")
    print(f"{name:18s} {dur:9.1f}us dram {rd:8.1f}+{wr:7.1f}MB "
          f"ipc {float(col(r, 'sm__inst_executed.avg.per_cycle_active') or 0):4.2f} "
          f"occ {float(col(r, 'sm__warps_active.avg.pct_of_peak_sustained_active') or 0):4.1f}% "
          f"inst {float(col(r, 'smsp__inst_executed.sum') or 0) / 1e6:7.1f}M  {st}")
