"""The paper's Leja-vs-Krylov comparison on one B200, config-1 state at N^2.

phi_1(dt J) v for alpha*dt in {1, 10, 100}, tol 1e-10, through the public API
with device tensors: iterations (= matvecs = RHS calls), device time per call,
and the two results' relative distance.  Also the MGS update kernel's
achieved bandwidth (32 B per element per update).

Usage: python scripts/krylov_vs_leja.py [n]   -> one JSON line per point
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13622_b200 as xb  # noqa: E402
from paper_2108_13622_b200 import leja, scenarios as sc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
s = sc.CONFIGS[1]()
s.nx = s.ny = n
q = sc.initial_fields(s)
st = xb.StateGrid(n, n, s.dx, s.dy, torch.from_numpy(q).cuda())
mhd = xb.MhdRhs(st, xb.MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa))
op = xb.RhsOperator(mhd)
lin = xb.FrozenLinearization(op, st.flat())
est = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0))
v = torch.from_numpy(sc.unit_gaussian(q.size, s.extra["v_seed"])).cuda()
mv = xb.JacobianAction(lin)


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0 = op.calls
    e0.record()
    res = fn()
    e1.record()
    torch.cuda.synchronize()
    return res, e0.elapsed_time(e1), op.calls - c0


for adt in (1.0, 10.0, 100.0):
    dt = adt / est.alpha
    leja._coeff_cache.clear()
    rl, tl, cl = timed(lambda: xb.apply_phi_leja(1, mv, v, dt, xb.shift_and_scale(adt), 1e-10))
    rk, tk, ck = timed(lambda: xb.apply_phi_krylov(1, mv, v, dt, 1e-10))
    d = float(torch.linalg.norm(rk.vector - rl.vector) / torch.linalg.norm(rl.vector))
    print(json.dumps({"n": n, "alpha": est.alpha, "adt": adt,
                      "leja": {"iterations": rl.iterations, "converged": rl.converged,
                               "rhs_calls": cl, "ms": tl},
                      "krylov": {"iterations": rk.iterations, "converged": rk.converged,
                                 "rhs_calls": ck, "ms": tk},
                      "krylov_over_leja_time": tk / tl, "rel_distance": d}), flush=True)

# MGS update kernel bandwidth: one Arnoldi step against 32 basis vectors
from paper_2108_13622_b200 import krylov  # noqa: E402
nb = 32
basis = [torch.randn(v.numel(), dtype=torch.float64, device="cuda") for _ in range(nb)]
w = torch.randn_like(v)
coef = np.zeros((2, nb))
h = xb.krylov._ops.util_ctx().bind_stream()
krylov._mgs_local(h, basis, w, coef)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 5
for _ in range(reps):
    krylov._mgs_local(h, basis, w, coef)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
launches = 2 * nb + 1
gbs = (32.0 * v.numel() * 2 * nb + 16.0 * v.numel()) / (ms * 1e-3) / 1e9
print(json.dumps({"mgs_step_nb": nb, "ms": ms, "launches": launches,
                  "ms_per_update": ms / launches, "gbs_algorithmic": gbs}), flush=True)
