"""Where the bench step's time goes besides the fused term: CUPTI timeline of
two config-1 sweeps (after warm-up), device busy time vs span, the idle gaps
between kernels and the per-kernel totals."""
import collections
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13622_b200 as xb  # noqa: E402
from paper_2108_13622_b200 import leja, scenarios as sc  # noqa: E402

s = sc.CONFIGS[1]()
q = sc.initial_fields(s)
u = torch.from_numpy(q).cuda().reshape(-1)
v = torch.from_numpy(sc.unit_gaussian(q.size, 2)).cuda()
st = xb.StateGrid(s.nx, s.ny, s.dx, s.dy, u.reshape(q.shape))
mhd = xb.MhdRhs(st, xb.MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa))
lin = xb.FrozenLinearization(xb.RhsOperator(mhd), u)
alpha = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0)).alpha
mv = xb.JacobianAction(lin)


def sweep():
    leja._coeff_cache.clear()
    for adt in (1.0, 10.0, 100.0, 300.0):
        dt = adt / alpha
        xb.apply_phi_leja(1, mv, v, dt, xb.shift_and_scale(alpha * dt), 1e-10)


for _ in range(3):
    sweep()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    sweep()
    sweep()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs), key=lambda x: x[0])
busy = sum(en - st for st, en, _ in ks)
span = ks[-1][1] - ks[0][0]
gaps = []
per = collections.defaultdict(lambda: [0, 0.0])
last = None
for st_, en, name in ks:
    short = name.split("(")[0].replace("void ", "")[:60]
    per[short][0] += 1
    per[short][1] += en - st_
    if last is not None and st_ > last[1]:
        gaps.append((st_ - last[1], last[2].split("(")[0][:40], short[:40]))
    last = (st_, en, name) if last is None or en > last[1] else last
print(f"2 sweeps: wall {wall*1e3:.1f} ms, device busy {busy/1e3:.1f} ms, span {span/1e3:.1f} ms, "
      f"idle {sum(g for g, _, _ in gaps)/1e3:.2f} ms in {len(gaps)} gaps")
agg = collections.defaultdict(lambda: [0, 0.0])
for g, a, b in gaps:
    agg[(a, b)][0] += 1
    agg[(a, b)][1] += g
for (a, b), (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:12]:
    print(f"  idle {t/1e3:8.3f} ms in {c:4d} gaps  {a} -> {b}")
for name, (c, t) in sorted(per.items(), key=lambda x: -x[1][1])[:12]:
    print(f"  {name:60s} {c:5d} {t/1e3:9.3f} ms avg {t/c:8.2f} us")
