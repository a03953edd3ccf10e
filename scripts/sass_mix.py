"""Dynamic SASS opcode mix + top stall lines from an ncu source-page CSV."""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ie = h.index("Instructions Executed")
src = h.index("Source")
st = h.index("Warp Stall Sampling (All Samples)")
mix = Counter()
stall = []
for r in rows[2:]:
    if len(r) <= ie:
        continue
    op = re.sub(r"^@!?U?P\w+\s+", "", r[src].strip()).split(" ")[0].split(".")[0]
    try:
        n = float(r[ie] or 0)
        s = float(r[st] or 0)
    except ValueError:
        continue
    mix[op] += n
    stall.append((s, r[0], r[src].strip()[:70]))
tot = sum(mix.values())
print(f"total warp-instructions {tot:.3e}")
for op, n in mix.most_common(30):
    print(f"  {op:10s} {n:12.3e} {100*n/tot:5.1f}%")
print("top stall lines:")
for s, a, t in sorted(stall, reverse=True)[:25]:
    print(f"  {s:8.0f} {a} {t}")
