"""Host time of the phases of a host-paced phi-action (4096^2): coefficient
chunk, start (uploads + init kernel enqueue), driver loop, result."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13622_b200 as xb  # noqa: E402
from paper_2108_13622_b200 import leja, scenarios as sc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
s = sc.kh_setup(n)
q = sc.initial_fields(s)
st = xb.StateGrid(n, n, s.dx, s.dy, torch.from_numpy(q).cuda())
mhd = xb.MhdRhs(st, xb.MHDParams(s.mu, s.eta, s.kappa))
lin = xb.FrozenLinearization(xb.RhsOperator(mhd), st.flat())
alpha = 5875.8 * (n / 2048.0) ** 2
T = {}


def wrap(mod, name):
    f = getattr(mod, name)

    def g(*a, **k):
        t0 = time.perf_counter()
        r = f(*a, **k)
        T.setdefault(name, []).append(time.perf_counter() - t0)
        return r
    setattr(mod, name, g)


for name in ("_newton_coeffs", "_start", "drive_fused"):
    wrap(leja, name)
v = lin.base_rhs
for k in range(12):
    adt = 2.0 + 0.37 * k
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = xb.apply_phi_leja(1, xb.JacobianAction(lin), v, adt / alpha, xb.shift_and_scale(adt), 1e-7)
    torch.cuda.synchronize()
    T.setdefault("call", []).append(time.perf_counter() - t0)
    T.setdefault("its", []).append(r.iterations)
for name, ts in T.items():
    if name == "its":
        print("iterations", ts)
    else:
        print(f"{name:16s} median {1e3 * float(np.median(ts[2:])):8.3f} ms   max {1e3 * max(ts[2:]):8.3f} ms")
