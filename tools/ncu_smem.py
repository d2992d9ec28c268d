"""Shared-memory instructions of one kernel in an ncu report: executed warp
instructions, wavefronts per instruction (and ideal), N-way conflicts, stall
share. Usage: ncu_smem.py REP KERNEL_REGEX [min_inst]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
mini = float(sys.argv[3]) if len(sys.argv) > 3 else 1e5
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


seen = set()
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot_s = sum(num(r[ix["Warp Stall Sampling (All Samples)"]]) for r in body)
tw = 0.0
print(f"{'sass':56} {'inst':>9} {'wf/i':>6} {'ideal':>6} {'nway':>6} {'stall%':>6}")
for r in body:
    key = r[ix["Address"]]
    if key in seen:
        continue
    seen.add(key)
    src = r[ix["Source"]].strip()
    if not any(k in src for k in ("LDS", "STS", "ATOMS", "REDS", "LDSM")):
        continue
    inst = num(r[ix["Instructions Executed"]])
    if inst < mini:
        continue
    wf = num(r[ix["L1 Wavefronts Shared"]])
    ide = num(r[ix["L1 Wavefronts Shared Ideal"]])
    nw = num(r[ix["L1 Conflicts Shared N-Way"]])
    st = num(r[ix["Warp Stall Sampling (All Samples)"]])
    tw += wf
    print(f"{src[:56]:56} {inst:9.3g} {wf / inst:6.2f} {ide / inst:6.2f} {nw / inst:6.2f} {100 * st / tot_s:6.1f}")
print("total shared wavefronts (listed):", f"{tw:.4g}")
