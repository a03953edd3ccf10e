"""Device timeline of an adaptive run (torch.profiler / CUPTI): kernel busy time
vs wall time, per-kernel totals, and the idle gaps between kernels.

usage: prof_timeline.py {c0|c2} [t_final] | {c3|c4} [steps]
"""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2108_13622_b200 as xb  # noqa: E402
from paper_2108_13622_b200 import leja, scenarios as sc  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c0"
tf = float(sys.argv[2]) if len(sys.argv) > 2 else None
if which in ("c3", "c4"):
    tf, steps = None, (int(sys.argv[2]) if len(sys.argv) > 2 else 5)
if which == "c4":
    s = sc.CONFIGS[4]()
    s.max_accepted = steps
    warm = sc.CONFIGS[4]()
    warm.max_accepted = 1
    scheme = xb.Scheme.EXPRB54S4
elif which == "c3":
    s = sc.CONFIGS[3]()
    s.max_accepted = steps
    warm = sc.kh_setup(4096, tol=1e-5, t_final=1e9, max_accepted=1)
    scheme = xb.Scheme.EXPRB43
elif which == "c0":
    s = sc.kh_setup(128) if tf is None else sc.kh_setup(128, t_final=tf)
    warm = sc.kh_setup(128, t_final=0.02)
    scheme = xb.Scheme.EXPRB43
else:
    s = sc.harris_setup(512) if tf is None else sc.harris_setup(512, t_final=tf)
    warm = sc.harris_setup(512, t_final=0.02)
    scheme = xb.Scheme.EXPRB54S4
xb.run(xb.RunConfig(scenario=warm, scheme=scheme, tol=s.tol, max_accepted=warm.max_accepted))
leja._coeff_cache.clear()
torch.cuda.synchronize()
acts = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
with torch.profiler.profile(activities=acts) as prof:
    t0 = time.perf_counter()
    rep = xb.run(xb.RunConfig(scenario=s, scheme=scheme, tol=s.tol, max_accepted=s.max_accepted))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs), key=lambda x: x[0])
busy = 0.0
last_end = None
gaps = []
per = collections.defaultdict(lambda: [0, 0.0])
for st, en, name in ks:
    busy += en - st
    key = name.replace("(anonymous namespace)::", "").split("(")[0][:70]
    per[key][0] += 1
    per[key][1] += en - st
    if last_end is not None:
        gaps.append(st - last_end)
    last_end = en if last_end is None else max(last_end, en)
span = (ks[-1][1] - ks[0][0]) if ks else 0
print(f"{which}: wall {wall*1e3:.2f} ms (profiled), {rep.accepted} steps, {rep.rhs_evals} rhs; "
      f"device events {len(ks)}, busy {busy/1e3:.2f} ms over span {span/1e3:.2f} ms")
gaps.sort()
if gaps:
    n = len(gaps)
    print(f"gaps: n={n} median {gaps[n//2]:.1f} us, p90 {gaps[int(n*0.9)]:.1f} us, "
          f"sum {sum(gaps)/1e3:.2f} ms, sum>20us {sum(g for g in gaps if g > 20)/1e3:.2f} ms")
big = []
prev = None
for st, en, name in ks:
    if prev is not None and st - prev[1] > 1000:
        big.append((st - prev[1], prev[2].split("(")[0][:50], name.split("(")[0][:50]))
    prev = (st, en, name) if prev is None or en > prev[1] else prev
for g, a, b in sorted(big, reverse=True)[:12]:
    print(f"  gap {g/1e3:8.2f} ms after {a} before {b}")
for name, (c, t) in sorted(per.items(), key=lambda x: -x[1][1])[:15]:
    print(f"  {name:60s} {c:6d} {t/1e3:9.3f} ms  avg {t/c:7.2f} us")
# steady state: the stepping phase (between the start-up pauses -- RNG draw, first
# estimate -- and the final checksum copy); idle time by the kernels around it
segs, cur_seg, prev_end = [], [], None
for st, en, name in ks:
    if prev_end is not None and st - prev_end > 2e5:
        segs.append(cur_seg)
        cur_seg = []
    cur_seg.append((st, en, name))
    prev_end = en if prev_end is None else max(prev_end, en)
segs.append(cur_seg)
# the stepping phase: the run without a 0.2 s pause that holds most Leja terms
tail = max(segs, key=lambda sg: sum('stencil_kernel<2' in k[2] for k in sg))
if len(tail) > 2:
    sspan = tail[-1][1] - tail[0][0]
    sbusy = sum(en - st for st, en, _ in tail)
    pairs = collections.defaultdict(lambda: [0, 0.0])
    pe, pn = tail[0][1], tail[0][2]
    for st, en, name in tail[1:]:
        g = st - pe
        if g > 5:
            key = (pn.replace("(anonymous namespace)::", "").split("(")[0][:34],
                   name.replace("(anonymous namespace)::", "").split("(")[0][:34])
            pairs[key][0] += 1
            pairs[key][1] += g
        if en > pe:
            pe, pn = en, name
    print(f"steady state: span {sspan/1e3:.1f} ms, busy {sbusy/1e3:.1f} ms, idle {(sspan-sbusy)/1e3:.1f} ms "
          f"({len(tail)} events)")
    for (a, b), (c, t) in sorted(pairs.items(), key=lambda x: -x[1][1])[:14]:
        print(f"  idle {t/1e3:8.2f} ms in {c:4d} gaps  after {a:34s} before {b}")
