"""ncu driver: the RHS and JVP stencil kernels at config-1 size, a few launches
each, no profiler of its own (CUPTI belongs to ncu).  Launch order: F(u) of
the linearization, then 3 x (RHS, JVP)."""
import os
import sys

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
lin = xb.FrozenLinearization(xb.RhsOperator(mhd), st.flat())
w = torch.from_numpy(sc.unit_gaussian(q.size, 2)).cuda()
for _ in range(3):
    mhd(st.flat())
    xb.jvp(lin, w)
torch.cuda.synchronize()
print("ok")
