"""Config-1 parity and rounding floor at full size (2048^2), per alpha*dt point.

SURVEY §8(c): per-call parity at config 1 is claimable only where the
problem's own rounding sensitivity allows it.  Per alpha*dt in
{1, 10, 100, 300} (tol 1e-10) this measures
  * GPU vs the CPU oracle (the reference's NumPy algorithm, bit-identical to
    it) at alpha*dt = 1 and 10, where the oracle finishes in minutes;
  * the rounding floor: GPU vs GPU with another work decomposition
    (XMHD_SEG_ROWS), i.e. another equally valid summation order of the norms
    -- the same kind of difference as OpenBLAS ddot vs a device reduction.
Bars: same iteration counts everywhere; GPU vs oracle <= 1e-10; the floor is
reported (gpurun_out/parity_c1.json, summarised in profiles/) and asserted
only at the low degrees.

Slow (several minutes of single-core NumPy): runs only with XMHD_C1_PARITY=1.
"""

import json
import os
import time

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(os.environ.get("XMHD_C1_PARITY") != "1",
                                 reason="set XMHD_C1_PARITY=1 (slow full-size parity run)")]

SWEEP = (1.0, 10.0, 100.0, 300.0)
TOL = 1e-10
N = int(os.environ.get("XMHD_C1_N", "2048"))


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _gpu_sweep(xb, s, q, v, seg=None):
    from paper_2108_13622_b200 import leja, mhd
    if seg is not None:
        os.environ["XMHD_SEG_ROWS"] = str(seg)
    try:
        mhd._ctx_cache.clear()
        st = xb.StateGrid(N, N, s.dx, s.dy, torch.from_numpy(q).cuda())
        op_mhd = xb.MhdRhs(st, xb.MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa))
        plan = op_mhd.ctx.plan()
    finally:
        os.environ.pop("XMHD_SEG_ROWS", None)
        mhd._ctx_cache.clear()
    lin = xb.FrozenLinearization(xb.RhsOperator(op_mhd), st.flat())
    est = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0))
    vd = torch.from_numpy(v).cuda()
    out = []
    for adt in SWEEP:
        leja._coeff_cache.clear()
        dt = adt / est.alpha
        res = xb.apply_phi_leja(1, xb.JacobianAction(lin), vd, dt,
                                xb.shift_and_scale(est.alpha * dt), TOL)
        out.append((res, res.vector.cpu().numpy()))
    return est.alpha, plan, out


def test_config1_parity_and_floor():
    import paper_2108_13622_b200 as xb
    from paper_2108_13622_b200 import scenarios as sc
    from oracle import leja_np as lj
    from oracle import mhd_np
    s = sc.CONFIGS[1]()
    s.nx = s.ny = N
    q = sc.initial_fields(s)
    v = sc.unit_gaussian(q.size, s.extra["v_seed"])

    alpha, plan, auto = _gpu_sweep(xb, s, q, v)
    alpha2, plan2, seg = _gpu_sweep(xb, s, q, v, seg=64)
    assert plan2 != plan

    def f(flat):
        return mhd_np.rhs(flat.reshape(q.shape), s.dx, s.dy, s.mu, s.eta, s.kappa)

    op = lj.CountedRhs(f)
    lin = lj.Frozen(op, q.reshape(-1).copy())
    report = {"n": N, "tol": TOL, "alpha": alpha, "alpha_seg64": alpha2, "plan": plan,
              "plan_seg64": plan2, "points": []}
    for adt, (ra, va), (rb, vb) in zip(SWEEP, auto, seg):
        pt = dict(adt=adt, iterations=ra.iterations, iterations_seg64=rb.iterations,
                  converged=ra.converged, floor_rel=_rel(vb, va))
        if adt <= 10.0:
            dt = adt / alpha
            qq, th = lj.shift_scale(alpha * dt)
            t0 = time.perf_counter()
            ro = lj.phi_leja(1, lambda w: lj.fd_jvp(lin, w), v, dt, qq, th, TOL,
                             lj.CoeffCache())
            pt.update(oracle_iterations=ro.iterations, oracle_seconds=time.perf_counter() - t0,
                      gpu_vs_oracle_rel=_rel(va, ro.vector))
        report["points"].append(pt)
        print(json.dumps(pt), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "parity_c1.json"), "w") as fh:
        json.dump(report, fh, indent=1)
    for pt in report["points"]:
        assert pt["iterations"] == pt["iterations_seg64"]
        if "gpu_vs_oracle_rel" in pt:
            assert pt["oracle_iterations"] == pt["iterations"]
            assert pt["gpu_vs_oracle_rel"] <= 1e-10
            assert pt["floor_rel"] <= 1e-10
