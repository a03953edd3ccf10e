"""Achieved HBM bandwidth of the streaming vector kernels (stage algebra, norms).

usage: prof_vec.py [n_side=4096]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2108_13622_b200 import _ops  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
n = 8 * side * side
peak = 6537.3
try:
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass
vs = [torch.randn(n, dtype=torch.float64, device="cuda") for _ in range(4)]
out = torch.empty_like(vs[0])


def timed(f, reps=10):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


cases = [
    ("lincomb2", 3, lambda: _ops.lincomb((1.0, 0.5), vs[:2], out=out)),
    ("lincomb3", 4, lambda: _ops.lincomb((1.0, 0.5, 0.25), vs[:3], out=out)),
    ("lincomb4", 5, lambda: _ops.lincomb((1.0, 0.5, 0.25, 2.0), vs[:4], out=out)),
    ("lincomb4+norm", 5, lambda: _ops.lincomb((1.0, 0.5, 0.25, 2.0), vs[:4], out=out, want_norm=True)),
    ("norm", 1, lambda: _ops.norm(vs[0])),
    ("diff_norms", 2, lambda: _ops.diff_norms(vs[0], vs[1])),
    ("divide", 2, lambda: _ops.divide(vs[0], 3.0, out=out)),
    ("torch add (ref)", 3, lambda: torch.add(vs[0], vs[1], out=out)),
    ("torch copy (ref)", 2, lambda: out.copy_(vs[0])),
]
for name, passes, f in cases:
    ms = timed(f)
    gbs = passes * n * 8 / (ms * 1e-3) / 1e9
    print(f"{name:18s} n={n} {ms:8.3f} ms  {gbs:7.0f} GB/s  {100 * gbs / peak:5.1f}% of HBM peak")
