"""Global-memory instructions of one kernel in an ncu report: executed warp
instructions, L1 tag requests, L2 theoretical sectors (and ideal) per SASS
load/store, plus stall samples. Usage: ncu_gmem.py REP KERNEL_REGEX"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot_s = sum(num(r[ix["Warp Stall Sampling (All Samples)"]]) for r in rows[2:] if len(r) == len(hdr))
print(f"{'sass':58} {'inst':>9} {'tagreq/i':>8} {'sect/i':>7} {'ideal/i':>7} {'stall%':>6}")
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    src = r[ix["Source"]].strip()
    if not any(k in src for k in ("LDG", "STG", "LD.", "ST.", "RED", "ATOM")) or "LDS" in src or "STS" in src:
        continue
    inst = num(r[ix["Instructions Executed"]])
    if inst == 0:
        continue
    tag = num(r[ix["L1 Tag Requests Global"]])
    sec = num(r[ix["L2 Theoretical Sectors Global"]])
    ide = num(r[ix["L2 Theoretical Sectors Global Ideal"]])
    st = num(r[ix["Warp Stall Sampling (All Samples)"]])
    print(f"{src[:58]:58} {inst:9.3g} {tag / inst:8.2f} {sec / inst:7.2f} {ide / inst:7.2f} {100 * st / tot_s:6.1f}")
