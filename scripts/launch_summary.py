"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel."""
import csv
import sys
from collections import defaultdict

rows = []
with open(sys.argv[1]) as fh:
    lines = [l for l in fh if l.startswith('"')]
rdr = csv.DictReader(lines)
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rdr:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    short = name.split("(")[0].replace("void ", "")
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
    tot[short] += v * scale
    cnt[short] += 1
allt = sum(tot.values())
print(f"# launch list summary ({sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]})")
print(f"# {sum(cnt.values())} launches, {allt/1e3:.2f} ms total device time (ncu: cold, serialised)")
print(f"{'kernel':70s} {'launches':>8s} {'total_us':>12s} {'share':>7s} {'avg_us':>9s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:70]:70s} {cnt[k]:8d} {tot[k]:12.1f} {100*tot[k]/allt:6.1f}% {tot[k]/cnt[k]:9.2f}")
