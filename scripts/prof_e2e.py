"""Break the bench e2e step (public API, pinned host buffers) into its parts."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13622_b200 as xb  # noqa: E402
from paper_2108_13622_b200 import leja, scenarios as sc  # noqa: E402

SWEEP = (1.0, 10.0, 100.0, 300.0)
s = sc.CONFIGS[1]()
q = sc.initial_fields(s)
v_host = sc.unit_gaussian(q.size, s.extra["v_seed"]).reshape(q.shape)
params = xb.MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa)
u_dev = torch.from_numpy(q).cuda().reshape(-1)
st = xb.StateGrid(s.nx, s.ny, s.dx, s.dy, u_dev.reshape(8, s.ny, s.nx))
mhd = xb.MhdRhs(st, params)
lin = xb.FrozenLinearization(xb.RhsOperator(mhd), u_dev)
alpha = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0)).alpha
u_pin = torch.from_numpy(q.reshape(-1)).pin_memory()
v_pin = torch.from_numpy(v_host.reshape(-1)).pin_memory()


def tick():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(3):
    leja._coeff_cache.clear()
    t0 = tick()
    lin_e = xb.FrozenLinearization(xb.RhsOperator(mhd), u_pin)
    t1 = tick()
    parts = []
    for adt in SWEEP:
        dt = adt / alpha
        a = tick()
        res = xb.apply_phi_leja(1, xb.JacobianAction(lin_e), v_pin, dt,
                                xb.shift_and_scale(alpha * dt), 1e-10)
        b = tick()
        parts.append((adt, res.iterations, round((b - a) * 1e3, 2)))
    print(f"rep {rep}: lin {1e3*(t1-t0):.2f} ms; phi calls (adt, its, ms) {parts}", flush=True)

# device-only reference for the same calls
for rep in range(2):
    leja._coeff_cache.clear()
    parts = []
    for adt in SWEEP:
        dt = adt / alpha
        a = tick()
        res = xb.apply_phi_leja(1, xb.JacobianAction(lin), torch.from_numpy(v_host.reshape(-1)).cuda(), dt,
                                xb.shift_and_scale(alpha * dt), 1e-10)
        b = tick()
        parts.append((adt, res.iterations, round((b - a) * 1e3, 2)))
    print(f"device rep {rep}: {parts}", flush=True)
