"""Split a kernel's SASS into barrier-delimited regions and report each region's
share of executed warp instructions and stall samples, plus the hottest
instructions (executed count, avg active threads). Usage:
ncu_regions.py REP KERNEL_REGEX [top_n]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ii, si, st, th = (hdr.index(k) for k in ("Instructions Executed", "Source",
                                        "Warp Stall Sampling (All Samples)", "Avg. Threads Executed"))
R = rows[2:]
tot = sum(float(r[ii]) for r in R)
stt = sum(float(r[st]) for r in R) or 1.0
print(f"total warp-inst {tot:.4g}")
cur, start = [0.0, 0.0], 0
for k, r in enumerate(R):
    cur[0] += float(r[ii])
    cur[1] += float(r[st])
    src = r[si].strip()
    if "BAR.SYNC" in src or "EXIT" in src or k == len(R) - 1:
        if cur[0] / tot > 0.01 or cur[1] / stt > 0.02:
            print(f"region {start:5d}-{k:5d}: inst {100 * cur[0] / tot:5.1f}%  stall {100 * cur[1] / stt:5.1f}%")
        cur, start = [0.0, 0.0], k + 1
items = sorted(((float(r[ii]), k, r) for k, r in enumerate(R)), reverse=True)[:top]
for v, k, r in sorted(items, key=lambda x: x[1]):
    print(f"{k:5d} {100 * v / tot:5.2f}% thr {float(r[th]):5.1f} stall {100 * float(r[st]) / stt:5.2f}%  {r[si].strip()[:70]}")
