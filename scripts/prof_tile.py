"""Per-term time of the one-launch Leja loop on small grids (CUDA events).

usage: prof_tile.py [n ...]   (XMHD_TILE=0: sliding-window loop)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13622_b200 as xb  # noqa: E402
from paper_2108_13622_b200 import leja, scenarios as sc  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [128, 512]:
    s = sc.harris_setup(n) if n == 512 else sc.kh_setup(n)
    q = sc.initial_fields(s)
    st = xb.StateGrid(n, n, s.dx, s.dy, torch.from_numpy(q).cuda())
    op = xb.RhsOperator(xb.MhdRhs(st, xb.MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa)))
    lin = xb.FrozenLinearization(op, st.flat())
    alpha = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0)).alpha
    v = torch.from_numpy(sc.unit_gaussian(q.size, 3)).cuda()
    for adt in (2.0, 20.0):
        sh = xb.shift_and_scale(adt)
        mv = xb.JacobianAction(lin)
        for _ in range(3):
            r = xb.apply_phi_leja(1, mv, v, adt / alpha, sh, 1e-10)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            r = xb.apply_phi_leja(1, mv, v, adt / alpha, sh, 1e-10)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"n={n} adt={adt}: {r.iterations} terms, {ms*1e3:.1f} us/call, "
              f"{ms*1e3/r.iterations:.2f} us/term", flush=True)
