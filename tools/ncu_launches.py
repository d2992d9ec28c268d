"""Per-kernel launch totals from an `ncu --metrics gpu__time_duration.sum --csv`
log (the B200_PROFILING launch-list pass). Usage: ncu_launches.py LOG [HEADER...]"""
import csv
import io
import sys
from collections import defaultdict

txt = open(sys.argv[1]).read()
start = txt.find('"ID"')
rows = list(csv.DictReader(io.StringIO(txt[start:])))
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "").strip()
    if len(name) > 34:
        name = name[:33] + "<"
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    v *= {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
    tot[name] += v
    cnt[name] += 1
S = sum(tot.values())
for h in sys.argv[2:]:
    print("# " + h)
print(f"{'kernel':<34} {'launches':>8} {'sum_ns':>12} {'share':>7}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:<34} {cnt[k]:>8} {tot[k]:>12.0f} {100 * tot[k] / S:>6.1f}%")
