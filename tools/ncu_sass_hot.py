"""Per-SASS-instruction hot spots of one kernel in an ncu report: executed warp
instructions, avg active threads, stall samples.
Usage: ncu_sass_hot.py REP KERNEL_REGEX [min_fraction]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
minf = float(sys.argv[3]) if len(sys.argv) > 3 else 0.004
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and "Source" in r and "Instructions Executed" in r)
ii, si, st, th = (hdr.index(k) for k in ("Instructions Executed", "Source",
                                        "Warp Stall Sampling (All Samples)", "Avg. Threads Executed"))


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


# SASS rows of the first listing only (the page may repeat the listing)
start = rows.index(hdr) + 1
R = []
for r in rows[start:]:
    if len(r) != len(hdr) or r[si] == "Source":
        break
    R.append(r)
tot = sum(num(r[ii]) for r in R) or 1.0
stot = sum(num(r[st]) for r in R) or 1.0
print(f"total warp-inst {tot:.4g}, stall samples {stot:.0f}")
for k, r in enumerate(R):
    v, s = num(r[ii]), num(r[st])
    if v / tot >= minf or s / stot >= 0.01:
        print(f"{k:5d} {100 * v / tot:5.2f}% thr {num(r[th]):5.1f} stall {100 * s / stot:5.2f}%  {r[si].strip()[:80]}")
