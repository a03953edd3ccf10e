"""Per-kind (odd PM_SKIP / even PM_LOOK) fused-term times for a given grid
and state (kh = config-1 state, harris = config-4 state): is the per-cell cost
a property of the size or of the state / division kinds?"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13622_b200 as xb  # noqa: E402
from paper_2108_13622_b200 import _lib, leja, scenarios as sc  # noqa: E402

n = int(sys.argv[1])
kind = sys.argv[2]
s = sc.CONFIGS[1]() if kind == "kh" else sc.CONFIGS[4]()
s.nx = s.ny = n
q = sc.initial_fields(s)
st = xb.StateGrid(n, n, s.dx, s.dy, torch.from_numpy(q).cuda())
mhd = xb.MhdRhs(st, xb.MHDParams(s.mu, s.eta, s.kappa))
lin = xb.FrozenLinearization(xb.RhsOperator(mhd), st.flat())
v = torch.from_numpy(sc.unit_gaussian(q.size, 2)).cuda()
alpha = 5875.8 * (n / 2048.0) ** 2 if kind == "kh" else 769.46 * (n / 8192.0) ** 2
dt = 10.0 / alpha
sh = xb.shift_and_scale(alpha * dt)
c = np.ascontiguousarray(leja._newton_coeffs(1, sh.q, sh.theta, 500))
xi = np.ascontiguousarray(leja.leja_points(500))
dp = ctypes.POINTER(ctypes.c_double)
out = ctypes.c_double()
kinds = (ctypes.c_double * 2)()
rc = _lib.load().xmhd_time_leja_iterations(mhd.ctx.bind_stream(), _lib.ptr(lin.base_state),
                                           _lib.ptr(lin.base_rhs), float(lin._base_norm),
                                           _lib.ptr(v), dt, sh.q, sh.theta, xi.ctypes.data_as(dp),
                                           c.ctypes.data_as(dp), 24, ctypes.byref(out), kinds)
assert rc == 0, _lib.err_text()
cells = n * n
print(f"{kind} {n}^2 plan {mhd.ctx.plan()} odd {kinds[0]:.4f} ms ({256*cells/kinds[0]/1e6:.0f} GB/s, "
      f"{kinds[0]*1e9/cells:.1f} ps/cell) even {kinds[1]:.4f} ms ({384*cells/kinds[1]/1e6:.0f} GB/s, "
      f"{kinds[1]*1e9/cells:.1f} ps/cell)")
