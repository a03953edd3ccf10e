"""Where the config-1 sweep step's device time goes beyond the fused kernel."""
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
st = xb.StateGrid(s.nx, s.ny, s.dx, s.dy, torch.from_numpy(q).cuda())
mhd = xb.MhdRhs(st, xb.MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa))
lin = xb.FrozenLinearization(xb.RhsOperator(mhd), st.flat())
alpha = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0)).alpha
v = torch.from_numpy(sc.unit_gaussian(q.size, s.extra["v_seed"])).cuda()
mv = xb.JacobianAction(lin)
for rep in range(4):
    leja._coeff_cache.clear()
    parts = []
    for adt in (1.0, 10.0, 100.0, 300.0):
        dt = adt / alpha
        torch.cuda.synchronize()
        l0 = mhd.ctx.launches()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        res = xb.apply_phi_leja(1, mv, v, dt, xb.shift_and_scale(alpha * dt), 1e-10)
        e1.record()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        parts.append((adt, res.iterations, round(e0.elapsed_time(e1), 2),
                      round((t1 - t0) * 1e3, 2), mhd.ctx.launches() - l0))
    print(f"rep {rep}: (adt, its, dev ms, wall ms, launches) {parts}", flush=True)
