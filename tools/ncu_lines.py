"""Aggregate an ncu source page (--print-source cuda,sass) per CUDA source line:
instructions executed and warp-stall samples. Usage: ncu_lines.py REP KERNEL_REGEX [N]"""
import csv, subprocess, sys, io

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, items, tot, stot = "", [], 0.0, 0.0
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ii = hdr.index("Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or not r or not r[0]:
        continue
    try:
        v, s = float(r[ii]), float(r[si])
    except (ValueError, IndexError):
        continue
    tot += v
    stot += s
    items.append((s, v, f"{fname}:{r[0]}", r[1].strip()[:90]))
items.sort(reverse=True)
print(f"total warp-inst {tot:.3g}  stall samples {stot:.0f}")
for s, v, loc, src in items[:n]:
    print(f"{100 * s / max(stot, 1):5.1f}% stall {100 * v / max(tot, 1):5.1f}% inst  {loc:24s} {src}")
