"""Device time of the RHS and JVP stencil kernels (CUPTI kernel durations via
torch.profiler; warm, back to back) at config-1 size, next to their
algorithmic bytes (RHS 128 B/cell: read u, write F; JVP 256 B/cell: read u,
w, F(u), write Jw) and fp64 operation counts."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13622_b200 as xb  # noqa: E402
from paper_2108_13622_b200 import scenarios as sc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
s = sc.CONFIGS[1]()
s.nx = s.ny = n
q = sc.initial_fields(s)
st = xb.StateGrid(n, n, s.dx, s.dy, torch.from_numpy(q).cuda())
mhd = xb.MhdRhs(st, xb.MHDParams(s.mu, s.eta, s.kappa))
op = xb.RhsOperator(mhd)
lin = xb.FrozenLinearization(op, st.flat())
w = torch.from_numpy(sc.unit_gaussian(q.size, 2)).cuda()
for _ in range(3):
    mhd(st.flat())
    xb.jvp(lin, w)
torch.cuda.synchronize()
acts = [torch.profiler.ProfilerActivity.CUDA]
with torch.profiler.profile(activities=acts) as prof:
    for _ in range(20):
        mhd(st.flat())
    for _ in range(20):
        xb.jvp(lin, w)
    torch.cuda.synchronize()
dur = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and "stencil" in e.name and "kernel<" in e.name:
        mode = e.name.split("kernel<", 1)[1][:1]
        key = "RHS" if mode == "0" else ("JVP" if mode == "1" else e.name)
        dur.setdefault(key, []).append(e.time_range.end - e.time_range.start)
cells = n * n
peak = 6529.7
for key, b in (("RHS", 128), ("JVP", 256)):
    d = np.median(dur[key])
    gbs = b * cells / (d * 1e-6) / 1e9
    print(f"n={n} {key}: {d:.1f} us median of {len(dur[key])}, {gbs:.0f} GB/s algorithmic "
          f"({b} B/cell) = {gbs / peak:.1%} of HBM peak", flush=True)
