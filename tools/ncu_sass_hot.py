"""Per-SASS-instruction hot spots of one kernel in an ncu report: executed warp
instructions, avg active threads, stall samples, with the CUDA source line.
Usage: ncu_sass_hot.py REP KERNEL_REGEX [min_fraction]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
minf = float(sys.argv[3]) if len(sys.argv) > 3 else 0.004
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, cur, items = None, "", []
for r in rows:
    if r and r[0] == "File Path":
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r:
        continue
    d = dict(zip(hdr, r))
    if r[0]:  # a CUDA source line
        cur = f"{r[0]}: {r[1].strip()[:60]}"
        continue
for r in rows:
    pass
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ii, si, st, th = (hdr.index(k) for k in ("Instructions Executed", "Source",
                                        "Warp Stall Sampling (All Samples)", "Avg. Threads Executed"))
R = rows[2:]
tot = sum(float(r[ii]) for r in R)
stot = sum(float(r[st]) for r in R)
print(f"total warp-inst {tot:.4g}, stall samples {stot:.0f}")
for k, r in enumerate(R):
    v, s = float(r[ii]), float(r[st])
    if v / tot >= minf or s / stot >= 0.01:
        print(f"{k:5d} {100 * v / tot:5.2f}% thr {float(r[th]):5.1f} stall {100 * s / stot:5.2f}%  {r[si].strip()[:80]}")
