"""Stall samples of one kernel split into the row-step phases of the sliding
window (the regions between BAR.SYNCs inside the hot loop).

usage: ncu -i REP --page source --csv --print-source sass --launch-skip K --launch-count 1 > x.csv
       python scripts/stall_regions.py x.csv
"""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
src = h.index("Source")
ie = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ri = [h.index(c) for c in reasons]
tot_i = h.index("Warp Stall Sampling (All Samples)")

region = 0
regs = {}
for r in rows[2:]:
    if len(r) <= ie:
        continue
    s = r[src].strip()
    op = re.sub(r"^@!?U?P\w+\s+", "", s).split(" ")[0]
    if op.startswith("BAR.SYNC"):
        region += 1
    d = regs.setdefault(region, {"n": 0.0, "samples": 0.0, "why": Counter(), "ops": Counter(),
                                 "first": r[0]})
    try:
        d["n"] += float(r[ie] or 0)
        d["samples"] += float(r[tot_i] or 0)
        for c, i in zip(reasons, ri):
            d["why"][c[6:]] += float(r[i] or 0)
        d["ops"][op.split(".")[0]] += float(r[ie] or 0)
    except ValueError:
        pass
tot = sum(d["samples"] for d in regs.values())
ntot = sum(d["n"] for d in regs.values())
for k, d in regs.items():
    if d["samples"] < 0.01 * tot:
        continue
    why = ", ".join(f"{w} {100 * v / d['samples']:.0f}%" for w, v in d["why"].most_common(5))
    ops = ", ".join(f"{o} {100 * v / max(d['n'], 1):.0f}%" for o, v in d["ops"].most_common(6))
    print(f"region {k} (from {d['first'][-6:]}): {100 * d['samples'] / tot:.1f}% of samples, "
          f"{100 * d['n'] / ntot:.1f}% of instructions\n   stalls: {why}\n   ops: {ops}")
