"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``xmhd`` from ``/root/reference/pkg/src`` (read-only) and stores the
reference's outputs on seeded BASELINE-style inputs under ``tests/golden/``.
The committed ``.npz`` files travel to the GPU box; ``/root/reference`` does not.
Nothing else in the repo reads ``/root/reference``.
"""

import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REPO)

import xmhd  # noqa: E402  (the reference)
from xmhd import harness as ref_harness  # noqa: E402
from xmhd import leja as ref_leja  # noqa: E402
from xmhd import linearize as ref_lin  # noqa: E402
from xmhd import phi as ref_phi  # noqa: E402
from xmhd.integrators import Scheme, step  # noqa: E402
from xmhd.mhd import Boundary, MHDParams, StateGrid, mhd_rhs  # noqa: E402
from xmhd.scenarios import Scenario  # noqa: E402

from paper_2108_13622_b200 import scenarios as sc  # noqa: E402

NV = 8


def bc(periodic):
    return Boundary.PERIODIC if periodic else Boundary.REFLECTING


def random_state(rng, nx, ny):
    q = 0.1 * rng.standard_normal((NV, ny, nx))
    q[0] = 1.0 + 0.1 * rng.standard_normal((ny, nx))
    q[7] = 6.0 + 0.1 * rng.standard_normal((ny, nx))
    return q


def setup_state(setup):
    return sc.initial_fields(setup)


def rhs_cases():
    rng = np.random.default_rng(11)
    cases = []
    kh = sc.kh_setup(32)
    cases.append(("kh32", setup_state(kh), kh.dx, kh.dy,
                  dict(mu=kh.mu, eta=kh.eta, kappa=kh.kappa), True, True))
    hs = sc.harris_setup(32)
    hs.ny = 24
    cases.append(("harris32x24", setup_state(hs), hs.dx, hs.dy,
                  dict(mu=hs.mu, eta=hs.eta, kappa=hs.kappa), True, True))
    km = sc.Setup(**{**sc.kh_setup(64).__dict__, "kind": "kh-modes", "nx": 33, "ny": 20,
                     "extra": {"mode_seed": 5}})
    cases.append(("khmodes33x20", setup_state(km), km.dx, km.dy,
                  dict(mu=km.mu, eta=km.eta, kappa=km.kappa), True, True))
    cases.append(("rand16x12_refl_y", random_state(rng, 16, 12), 0.1, 0.15,
                  dict(mu=0.03, eta=0.02, kappa=0.1), True, False))
    cases.append(("rand20x16_refl_xy_mu0", random_state(rng, 20, 16), 0.07, 0.11,
                  dict(mu=0.05, eta=0.01, kappa=0.2, gamma=1.4, mu0=1.3), False, False))
    cases.append(("rand16x16_ideal", random_state(rng, 16, 16), 0.1, 0.1,
                  dict(mu=0.0, eta=0.0, kappa=0.0), True, True))
    cases.append(("rand17x9_refl_x", random_state(rng, 17, 9), 0.05, 0.2,
                  dict(mu=0.02, eta=0.0, kappa=0.0), False, True))
    cases.append(("tiny3x4", random_state(rng, 3, 4), 0.3, 0.25,
                  dict(mu=0.01, eta=0.02, kappa=0.03), True, True))
    cases.append(("rand200x5", random_state(rng, 200, 5), 0.01, 0.02,
                  dict(mu=0.01, eta=0.02, kappa=0.03), True, True))
    out = {}
    meta = []
    for name, q, dx, dy, prm, px, py in cases:
        params = MHDParams(bc_x=bc(px), bc_y=bc(py), **prm)
        f = mhd_rhs(StateGrid(q.shape[2], q.shape[1], dx, dy, q.copy()), params)
        out[f"{name}__u"] = q
        out[f"{name}__f"] = f
        meta.append(dict(name=name, dx=dx, dy=dy, periodic_x=px, periodic_y=py,
                         mu=params.mu, eta=params.eta, kappa=params.kappa,
                         gamma=params.gamma, mu0=params.mu0))
    # non-finite detection (mhd.py:225-231): zero density in one cell
    q = random_state(rng, 16, 12)
    q[0, 4, 5] = 0.0
    q[0, 9, 2] = 0.0
    params = MHDParams(mu=0.01, eta=0.01, kappa=0.01)
    try:
        mhd_rhs(StateGrid(16, 12, 0.1, 0.1, q.copy()), params)
        raise RuntimeError("expected RhsBlowupError")
    except ref_lin.RhsBlowupError as err:
        out["blowup__u"] = q
        meta.append(dict(name="blowup", dx=0.1, dy=0.1, periodic_x=True, periodic_y=True,
                         mu=0.01, eta=0.01, kappa=0.01, gamma=params.gamma, mu0=1.0,
                         cells=err.cells, message=str(err)))
    np.savez_compressed(os.path.join(HERE, "rhs_cases.npz"), **out)
    return meta


def mhd_op(q, dx, dy, params):
    g = StateGrid(q.shape[2], q.shape[1], dx, dy, q.copy())
    return ref_lin.RhsOperator(lambda flat: mhd_rhs(g.with_flat(flat), params))


def leja_cases():
    out = {}
    meta = []
    for tag, setup in (("kh32", sc.kh_setup(32)),
                       ("harris32", sc.harris_setup(32)),
                       ("khmodes48", sc.Setup(**{**sc.kh_setup(48).__dict__,
                                                  "kind": "kh-modes",
                                                  "extra": {"mode_seed": 3}}))):
        q = setup_state(setup)
        params = MHDParams(mu=setup.mu, eta=setup.eta, kappa=setup.kappa)
        op = mhd_op(q, setup.dx, setup.dy, params)
        u = q.reshape(-1).copy()
        lin = ref_lin.FrozenLinearization(op, u)
        before_power = op.calls
        est = ref_lin.estimate_alpha(lin, None, rng=np.random.default_rng(0))
        power_calls = op.calls - before_power
        out[f"{tag}__u"] = q
        out[f"{tag}__fu"] = lin.base_rhs
        out[f"{tag}__power_vec"] = est.vector
        w = sc.unit_gaussian(u.size, 7)
        out[f"{tag}__w"] = w
        out[f"{tag}__jw"] = ref_lin.jvp(lin, w)
        rec = dict(name=tag, dx=setup.dx, dy=setup.dy, mu=setup.mu, eta=setup.eta,
                   kappa=setup.kappa, alpha=est.alpha, power_calls=power_calls,
                   phi=[])
        v = sc.unit_gaussian(u.size, 8)
        out[f"{tag}__v"] = v
        for l in (0, 1, 3, 4):
            for adt in (1.0, 10.0):
                if tag != "kh32" and l in (0, 3):
                    continue
                dt = adt / est.alpha
                shift = ref_leja.shift_and_scale(est.alpha * dt)
                ref_leja._coeff_cache.clear()
                before = op.calls
                res = ref_leja.apply_phi_leja(l, lambda x: ref_lin.jvp(lin, x), v, dt,
                                              shift, 1e-10)
                key = f"{tag}__phi_l{l}_a{adt:g}"
                out[key] = res.vector
                rec["phi"].append(dict(key=key, l=l, adt=adt, dt=dt, q=shift.q,
                                       theta=shift.theta, tol=1e-10,
                                       iterations=res.iterations,
                                       converged=res.converged,
                                       residual=res.residual,
                                       rhs_calls=op.calls - before))
        meta.append(rec)
    np.savez_compressed(os.path.join(HERE, "leja_cases.npz"), **out)
    return meta


def leja_bc_cases():
    """JVP, power iteration and phi on reflecting walls, mu0 != 1, gamma != 5/3 and
    non-power-of-two spacings (the Markstein division paths of the kernels)."""
    out = {}
    meta = []
    rng = np.random.default_rng(21)
    for tag, nx, ny, dx, dy, px, py, prm in (
            ("rand40x28_refl_xy", 40, 28, 0.07, 0.11, False, False,
             dict(mu=0.02, eta=0.01, kappa=0.05, gamma=1.4, mu0=1.3)),
            ("rand36x30_refl_y", 36, 30, 0.1, 0.15, True, False,
             dict(mu=0.01, eta=0.02, kappa=0.03)),
            ("rand33x21_refl_x_ideal", 33, 21, 0.05, 0.2, False, True,
             dict(mu=0.0, eta=0.0, kappa=0.0))):
        q = random_state(rng, nx, ny)
        params = MHDParams(bc_x=bc(px), bc_y=bc(py), **prm)
        op = mhd_op(q, dx, dy, params)
        u = q.reshape(-1).copy()
        lin = ref_lin.FrozenLinearization(op, u)
        before = op.calls
        est = ref_lin.estimate_alpha(lin, None, rng=np.random.default_rng(0))
        power_calls = op.calls - before
        w = sc.unit_gaussian(u.size, 7)
        out[f"{tag}__u"] = q
        out[f"{tag}__fu"] = lin.base_rhs
        out[f"{tag}__w"] = w
        out[f"{tag}__jw"] = ref_lin.jvp(lin, w)
        out[f"{tag}__power_vec"] = est.vector
        v = sc.unit_gaussian(u.size, 8)
        out[f"{tag}__v"] = v
        rec = dict(name=tag, dx=dx, dy=dy, periodic_x=px, periodic_y=py, mu=params.mu,
                   eta=params.eta, kappa=params.kappa, gamma=params.gamma, mu0=params.mu0,
                   alpha=est.alpha, power_calls=power_calls, phi=[])
        for l, adt in ((1, 1.0), (1, 10.0), (4, 10.0), (0, 3.0)):
            dt = adt / est.alpha
            shift = ref_leja.shift_and_scale(est.alpha * dt)
            ref_leja._coeff_cache.clear()
            before = op.calls
            res = ref_leja.apply_phi_leja(l, lambda x: ref_lin.jvp(lin, x), v, dt, shift, 1e-10)
            key = f"{tag}__phi_l{l}_a{adt:g}"
            out[key] = res.vector
            rec["phi"].append(dict(key=key, l=l, adt=adt, dt=dt, q=shift.q, theta=shift.theta,
                                   tol=1e-10, iterations=res.iterations,
                                   converged=res.converged, residual=res.residual,
                                   rhs_calls=op.calls - before))
        meta.append(rec)
    np.savez_compressed(os.path.join(HERE, "leja_bc_cases.npz"), **out)
    return meta


def coeff_cases():
    out = {"leja_points": np.asarray(ref_leja.leja_points(500))}
    meta = []
    for l, alpha_dt, count in ((0, 1.0, 64), (1, 1.0, 64), (1, 10.0, 128), (3, 30.0, 256),
                               (4, 100.0, 500), (1, 300.0, 500), (2, 0.01, 64)):
        sh = ref_leja.shift_and_scale(alpha_dt)
        ref_leja._coeff_cache.clear()
        c = ref_leja._newton_coeffs(l, sh.q, sh.theta, count)
        key = f"coeff_l{l}_adt{alpha_dt:g}_n{count}"
        out[key] = c
        meta.append(dict(key=key, l=l, q=sh.q, theta=sh.theta, count=count))
    nodes = np.asarray(ref_leja.leja_points(64))
    for l in (0, 1, 3):
        out[f"divdiff_l{l}"] = ref_phi.divided_differences(l, nodes).coeffs
    np.savez_compressed(os.path.join(HERE, "coeff_cases.npz"), **out)
    return meta


def step_cases():
    out = {}
    meta = []
    for tag, setup, scheme, dt in (("kh32_exprb43", sc.kh_setup(32), Scheme.EXPRB43, 2e-3),
                                   ("harris32_exprb54s4", sc.harris_setup(32),
                                    Scheme.EXPRB54S4, 0.05),
                                   ("kh32_epirk5p1", sc.kh_setup(32), Scheme.EPIRK5P1, 2e-3),
                                   ("kh32_rosEuler", sc.kh_setup(32), Scheme.ROS_EULER, 1e-3),
                                   ("kh32_rk43", sc.kh_setup(32), Scheme.RK43, 1e-4),
                                   ("harris32_dopri54", sc.harris_setup(32), Scheme.DOPRI54,
                                    0.01)):
        q = setup_state(setup)
        params = MHDParams(mu=setup.mu, eta=setup.eta, kappa=setup.kappa)
        op = mhd_op(q, setup.dx, setup.dy, params)
        u = q.reshape(-1).copy()
        lin = ref_lin.FrozenLinearization(op, u)
        est = ref_lin.estimate_alpha(lin, None, rng=np.random.default_rng(0))
        ref_leja._coeff_cache.clear()
        before = op.calls
        res = step(scheme, op, u, dt, method="leja", alpha=est, tol=setup.tol, lin=lin)
        out[f"{tag}__u"] = q
        out[f"{tag}__new"] = res.new_state
        meta.append(dict(name=tag, scheme=scheme.value, dt=dt, tol=setup.tol,
                         alpha=est.alpha, error=res.error_estimate,
                         rhs_calls=res.rhs_calls, step_calls=op.calls - before,
                         phi_iterations=res.phi_iterations,
                         phi_applications=res.phi_applications,
                         converged=res.converged, dx=setup.dx, dy=setup.dy,
                         mu=setup.mu, eta=setup.eta, kappa=setup.kappa))
    np.savez_compressed(os.path.join(HERE, "step_cases.npz"), **out)
    return meta


def run_case(setup, scheme, method="leja"):
    q = setup_state(setup)
    params = MHDParams(mu=setup.mu, eta=setup.eta, kappa=setup.kappa)
    spec = Scenario(problem="custom", case_id=setup.name, nx=setup.nx, ny=setup.ny,
                    t_final=setup.t_final, x_min=setup.x_min, x_max=setup.x_max,
                    y_min=setup.y_min, y_max=setup.y_max, params=params, tol=setup.tol)
    state0 = StateGrid(setup.nx, setup.ny, setup.dx, setup.dy, q.copy())
    saved = ref_harness.initialize
    ref_harness.initialize = lambda _spec: StateGrid(state0.nx, state0.ny, state0.dx,
                                                      state0.dy, state0.data.copy())
    ref_leja._coeff_cache.clear()
    try:
        t0 = time.perf_counter()
        rep = ref_harness.run(ref_harness.RunConfig(scenario=spec, scheme=scheme,
                                                    method=method, tol=setup.tol,
                                                    rng_seed=setup.seed))
        wall = time.perf_counter() - t0
    finally:
        ref_harness.initialize = saved
    recs = [dict(t=s.t, dt=s.dt, error=s.error, rhs_calls=s.rhs_calls,
                 phi_iterations=s.phi_iterations, phi_applications=s.phi_applications,
                 accepted=s.accepted, cost=s.cost) for s in rep.steps]
    meta = dict(name=setup.name, nx=setup.nx, ny=setup.ny, scheme=scheme.value,
                tol=setup.tol, t_final=setup.t_final, accepted=rep.accepted,
                rejected=rep.rejected, rhs_evals=rep.rhs_evals,
                phi_iterations=rep.phi_iterations,
                spectrum_rhs_evals=rep.spectrum_rhs_evals, status=rep.status,
                checksum=rep.checksum, max_divb=rep.max_divb,
                mass_drift=rep.mass_drift, t_reached=rep.t_reached, steps=recs,
                wall_seconds=wall)
    return meta, rep.final_state.data


def run_cases():
    out = {}
    meta = []
    c0 = sc.kh_setup(128)
    m, fin = run_case(c0, Scheme.EXPRB43)
    out["C0__final"] = fin
    meta.append(m)
    h = sc.harris_setup(64, t_final=1.0, name="C2_64_t1")
    m, fin = run_case(h, Scheme.EXPRB54S4)
    out["C2_64_t1__final"] = fin
    meta.append(m)
    k = sc.kh_setup(32, t_final=0.2, name="C0_32_t0.2")
    m, fin = run_case(k, Scheme.EXPRB43)
    out["C0_32_t0.2__final"] = fin
    meta.append(m)
    np.savez_compressed(os.path.join(HERE, "run_cases.npz"), **out)
    return meta


def krylov_cases():
    """The Krylov baseline (krylov.py) on the fused-JVP matvec, a Krylov step and run."""
    from xmhd.krylov import apply_phi_krylov
    out = {}
    meta = {"phi": [], "step": [], "run": []}
    for tag, setup in (("kh32", sc.kh_setup(32)), ("harris32", sc.harris_setup(32))):
        q = setup_state(setup)
        params = MHDParams(mu=setup.mu, eta=setup.eta, kappa=setup.kappa)
        op = mhd_op(q, setup.dx, setup.dy, params)
        u = q.reshape(-1).copy()
        lin = ref_lin.FrozenLinearization(op, u)
        est = ref_lin.estimate_alpha(lin, None, rng=np.random.default_rng(0))
        v = sc.unit_gaussian(u.size, 8)
        out[f"{tag}__u"] = q
        out[f"{tag}__v"] = v
        cases = [(1, 1.0, 1e-10, 100), (1, 10.0, 1e-10, 100), (0, 10.0, 1e-8, 100),
                 (4, 10.0, 1e-8, 100), (2, 3.0, 1e-12, 100), (1, 10.0, 1e-10, 5)]
        if tag != "kh32":
            cases = cases[:2]
        for l, adt, tol, m_max in cases:
            dt = adt / est.alpha
            before = op.calls
            res = apply_phi_krylov(l, lambda x: ref_lin.jvp(lin, x), v, dt, tol, m_max)
            key = f"{tag}__kry_l{l}_a{adt:g}_t{tol:g}_m{m_max}"
            out[key] = res.vector
            meta["phi"].append(dict(key=key, case=tag, l=l, adt=adt, dt=dt, tol=tol,
                                    m_max=m_max, alpha=est.alpha, iterations=res.iterations,
                                    converged=res.converged, residual=res.residual,
                                    rhs_calls=op.calls - before, dx=setup.dx, dy=setup.dy,
                                    mu=setup.mu, eta=setup.eta, kappa=setup.kappa))
    for tag, setup, scheme, dt in (("kh32_exprb43_krylov", sc.kh_setup(32), Scheme.EXPRB43,
                                    2e-3),
                                   ("harris32_exprb54s4_krylov", sc.harris_setup(32),
                                    Scheme.EXPRB54S4, 0.05)):
        q = setup_state(setup)
        params = MHDParams(mu=setup.mu, eta=setup.eta, kappa=setup.kappa)
        op = mhd_op(q, setup.dx, setup.dy, params)
        u = q.reshape(-1).copy()
        lin = ref_lin.FrozenLinearization(op, u)
        est = ref_lin.estimate_alpha(lin, None, rng=np.random.default_rng(0))
        before = op.calls
        res = step(scheme, op, u, dt, method="krylov", alpha=est, tol=setup.tol, lin=lin)
        out[f"{tag}__u"] = q
        out[f"{tag}__new"] = res.new_state
        meta["step"].append(dict(name=tag, scheme=scheme.value, dt=dt, tol=setup.tol,
                                 alpha=est.alpha, error=res.error_estimate,
                                 rhs_calls=res.rhs_calls, step_calls=op.calls - before,
                                 phi_iterations=res.phi_iterations,
                                 phi_applications=res.phi_applications,
                                 converged=res.converged, dx=setup.dx, dy=setup.dy,
                                 mu=setup.mu, eta=setup.eta, kappa=setup.kappa))
    k = sc.kh_setup(32, t_final=0.2, name="C0_32_t0.2_krylov")
    m, fin = run_case(k, Scheme.EXPRB43, method="krylov")
    out["C0_32_t0.2_krylov__final"] = fin
    meta["run"].append(m)
    np.savez_compressed(os.path.join(HERE, "krylov_cases.npz"), **out)
    return meta


def wp_cases():
    """make_reference + work_precision (harness.py:255-327) on a small KH grid."""
    import tempfile
    from dataclasses import replace
    setup = sc.kh_setup(32, t_final=0.1, name="wp32")
    q = setup_state(setup)
    params = MHDParams(mu=setup.mu, eta=setup.eta, kappa=setup.kappa)
    spec = Scenario(problem="custom", case_id=setup.name, nx=setup.nx, ny=setup.ny,
                    t_final=setup.t_final, x_min=setup.x_min, x_max=setup.x_max,
                    y_min=setup.y_min, y_max=setup.y_max, params=params, tol=setup.tol)
    state0 = StateGrid(setup.nx, setup.ny, setup.dx, setup.dy, q.copy())
    saved = ref_harness.initialize
    ref_harness.initialize = lambda _spec: StateGrid(state0.nx, state0.ny, state0.dx,
                                                      state0.dy, state0.data.copy())
    ref_leja._coeff_cache.clear()
    out = {}
    try:
        base = ref_harness.RunConfig(scenario=spec, rng_seed=setup.seed)
        with tempfile.TemporaryDirectory() as tmp:
            ref_path = os.path.join(tmp, "ref.chk")
            rep = ref_harness.make_reference(base, ref_path)
            out["reference_final"] = rep.final_state.data
            out["reference_chk"] = np.frombuffer(open(ref_path, "rb").read(), dtype=np.uint8)
            rows = ref_harness.work_precision(base, [1e-3, 1e-5], [Scheme.EXPRB43,
                                                                   Scheme.EXPRB54S4],
                                              ["leja", "krylov"], ref_path,
                                              os.path.join(tmp, "wp.csv"))
            series, srep = ref_harness.divb_series(replace(base, tol=1e-4), 0.02)
    finally:
        ref_harness.initialize = saved
    keep = [{k: v for k, v in r.items() if k not in ("wall_seconds", "timestamp")}
            for r in rows]
    np.savez_compressed(os.path.join(HERE, "wp_cases.npz"), **out)
    return dict(setup=dict(nx=setup.nx, t_final=setup.t_final, seed=setup.seed),
                reference=dict(accepted=rep.accepted, rejected=rep.rejected,
                               rhs_evals=rep.rhs_evals, t_reached=rep.t_reached),
                rows=keep, divb_series=[[float(t), float(v)] for t, v in series],
                divb_accepted=srep.accepted)


def main():
    which = sys.argv[1:] or ["rhs", "leja", "leja_bc", "coeff", "step", "run", "krylov", "wp"]
    path = os.path.join(HERE, "golden_meta.json")
    meta = json.load(open(path)) if os.path.exists(path) else {}
    meta["generator"] = "tests/golden/make_golden.py (reference xmhd %s, numpy %s)" % (
        xmhd.__version__, np.__version__)
    fns = dict(rhs=rhs_cases, leja=leja_cases, coeff=coeff_cases, step=step_cases,
               run=run_cases, krylov=krylov_cases, wp=wp_cases, leja_bc=leja_bc_cases)
    for w in which:
        t0 = time.perf_counter()
        meta[w] = fns[w]()
        print(f"{w}: {time.perf_counter() - t0:.1f}s", flush=True)
    with open(path, "w") as fh:
        json.dump(meta, fh, indent=1, default=float)


if __name__ == "__main__":
    main()
