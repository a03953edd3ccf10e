"""Per-call wall/device split of the bench's config-1 sweep step (host coefficient
time vs device time), to explain a slow bench `value`.

usage: diag_sweep.py [steps]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13622_b200 as xb  # noqa: E402
from paper_2108_13622_b200 import leja, scenarios as sc  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
s = sc.CONFIGS[1]()
q = sc.initial_fields(s)
st = xb.StateGrid(s.nx, s.ny, s.dx, s.dy, torch.from_numpy(q).cuda())
mhd = xb.MhdRhs(st, xb.MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa))
lin = xb.FrozenLinearization(xb.RhsOperator(mhd), st.flat())
alpha = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0)).alpha
v = torch.from_numpy(sc.unit_gaussian(q.size, s.extra["v_seed"])).cuda()
mv = xb.JacobianAction(lin)

orig = leja._newton_coeffs
coef_s = []


def timed(*a, **k):
    t0 = time.perf_counter()
    r = orig(*a, **k)
    coef_s.append(time.perf_counter() - t0)
    return r


leja._newton_coeffs = timed
for step in range(steps):
    leja._coeff_cache.clear()
    rows = []
    torch.cuda.synchronize()
    for adt in (1.0, 10.0, 100.0, 300.0):
        coef_s.clear()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        r = xb.apply_phi_leja(1, mv, v, adt / alpha, xb.shift_and_scale(alpha * adt / alpha), 1e-10)
        e1.record()
        torch.cuda.synchronize()
        rows.append({"adt": adt, "terms": r.iterations, "wall_ms": round(1e3 * (time.perf_counter() - t0), 2),
                     "event_ms": round(e0.elapsed_time(e1), 2),
                     "coeff_ms": [round(1e3 * c, 2) for c in coef_s]})
    print(json.dumps({"step": step, "calls": rows}), flush=True)
