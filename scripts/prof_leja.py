"""Small driver for ncu: config-1 state at N^2, one F(u), then the fused Leja
iteration kernel back-to-back (xmhd_time_leja_iterations).  Kernel order:
stencil<RHS> (F(u)), norm, leja_init, stencil<LEJA> warm-up, stencil<LEJA> x n."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13622_b200 as xb  # noqa: E402
from paper_2108_13622_b200 import _lib, leja, scenarios as sc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
s = sc.CONFIGS[1]()
s.nx = s.ny = n
q = sc.initial_fields(s)
st = xb.StateGrid(n, n, s.dx, s.dy, torch.from_numpy(q).cuda())
mhd = xb.MhdRhs(st, xb.MHDParams(s.mu, s.eta, s.kappa))
lin = xb.FrozenLinearization(xb.RhsOperator(mhd), st.flat())
v = torch.from_numpy(sc.unit_gaussian(q.size, 2)).cuda()
alpha = 5875.8 * (n / 2048.0) ** 2
dt = 10.0 / alpha
sh = xb.shift_and_scale(alpha * dt)
c = np.ascontiguousarray(leja._newton_coeffs(1, sh.q, sh.theta, 500))
xi = np.ascontiguousarray(leja.leja_points(500))
dp = ctypes.POINTER(ctypes.c_double)
out = ctypes.c_double()
rc = _lib.load().xmhd_time_leja_iterations(mhd.ctx.bind_stream(), _lib.ptr(lin.base_state),
                                           _lib.ptr(lin.base_rhs), float(lin._base_norm),
                                           _lib.ptr(v), dt, sh.q, sh.theta, xi.ctypes.data_as(dp),
                                           c.ctypes.data_as(dp), iters, ctypes.byref(out), None)
assert rc == 0, _lib.err_text()
torch.cuda.synchronize()
print(mhd.ctx.plan())
print(f"n={n} fused Leja iteration: {out.value:.4f} ms -> "
      f"{384 * n * n / (out.value * 1e-3) / 1e9:.1f} GB/s algorithmic")
