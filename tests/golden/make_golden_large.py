"""Golden fixtures at the BENCHMARKED sizes, produced by the REFERENCE itself.

Run in the build container (where /root/reference exists), one job per
process (they are long; run them side by side):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_large.py c1-alpha
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_large.py c1-point 300
    OPENBLAS_NUM_THREADS=8 python tests/golden/make_golden_large.py c1-point 300
    ...                                                   (adt in 1 10 100 300)
    python tests/golden/make_golden_large.py c1-combine
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_large.py degree
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_large.py c2
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_large.py c3
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_large.py c4

Everything is computed by ``xmhd`` from ``/root/reference/pkg/src`` (read
only) on the seeded BASELINE inputs of ``paper_2108_13622_b200.scenarios``.
Vectors at these sizes are 0.27-4.3 GB, so the fixtures keep what a test
needs to compare against: iteration / step / RHS counters, scalar results,
exact norms and strided samples of the result vectors, plus the sha256 of the
inputs so the GPU test can prove it rebuilt the same inputs on its host.

Parity floors: the reference's own result depends on the
summation order of ``np.linalg.norm`` (OpenBLAS ``ddot`` splits a vector over
its threads).  The "floor" of a configuration is the relative L2 distance
between two reference runs that differ only in that order (1 vs 8 BLAS
threads at 2048^2; a correctly rounded ``math.fsum`` norm at the small sizes
where ``ddot`` does not thread).  A GPU result is held to max(bar, floor-based
bound) where the test says so.

Outputs go to ``tests/golden/large/`` (one ``.json`` + ``.npz`` per case);
the full 2048^2 vectors of the floor runs are kept in /tmp only.
"""

import hashlib
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "large")
SCRATCH = "/tmp/xmhd_golden_large"
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REPO)

import xmhd  # noqa: E402  (the reference)
from xmhd import harness as ref_harness  # noqa: E402
from xmhd import leja as ref_leja  # noqa: E402
from xmhd import linearize as ref_lin  # noqa: E402
from xmhd.integrators import Scheme  # noqa: E402
from xmhd.mhd import MHDParams, StateGrid, mhd_rhs  # noqa: E402
from xmhd.scenarios import Scenario  # noqa: E402

from paper_2108_13622_b200 import scenarios as sc  # noqa: E402

C1_SWEEP = (1.0, 10.0, 100.0, 300.0)
C1_TOL = 1e-10
C1_STRIDE = 389          # strided sample of the 33.5 M-entry phi result (86 k values)
C3_STRIDE = 61           # 134 M-entry state -> 2.2 M values
C2_STRIDE = 4            # 2.1 M-entry state -> 524 k values
C4_COL_STRIDE = 8


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def blas_threads():
    return int(os.environ.get("OPENBLAS_NUM_THREADS", "0") or 0)


def save(name, meta, arrays=None):
    os.makedirs(OUT, exist_ok=True)
    meta = dict(meta, generator="tests/golden/make_golden_large.py (reference xmhd %s, numpy %s)"
                % (xmhd.__version__, np.__version__))
    with open(os.path.join(OUT, name + ".json"), "w") as fh:
        json.dump(meta, fh, indent=1, default=float)
    if arrays:
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrays)


def mhd_op(q, dx, dy, params):
    g = StateGrid(q.shape[2], q.shape[1], dx, dy, q.copy())
    return ref_lin.RhsOperator(lambda flat: mhd_rhs(g.with_flat(flat), params))


# ---------------------------------------------------------------- config 1

def c1_inputs():
    s = sc.CONFIGS[1]()
    q = sc.initial_fields(s)
    v = sc.unit_gaussian(q.size, s.extra["v_seed"])
    params = MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa)
    return s, q, v, params


def c1_alpha():
    """alpha of the config-1 state: the reference's power iteration, start
    vector from default_rng(0) as the bench and the GPU test use."""
    s, q, v, params = c1_inputs()
    op = mhd_op(q, s.dx, s.dy, params)
    lin = ref_lin.FrozenLinearization(op, q.reshape(-1).copy())
    before = op.calls
    t0 = time.perf_counter()
    est = ref_lin.estimate_alpha(lin, None, rng=np.random.default_rng(0))
    sec = time.perf_counter() - t0
    fu = lin.base_rhs
    save("c1_alpha", dict(n=s.nx, alpha=est.alpha, power_calls=op.calls - before,
                          power_seconds=sec, unorm=lin._base_norm, u_sha256=sha(q),
                          v_sha256=sha(v), fu_norm=float(np.sqrt(np.add.reduce(fu * fu))),
                          fu_sha256=sha(fu), blas_threads=blas_threads(),
                          stride=C1_STRIDE),
         dict(fu_sample=fu[::C1_STRIDE]))


def c1_point(adt):
    """One phi_1 call of the config-1 sweep at alpha*dt = adt (tol 1e-10)."""
    adt = float(adt)
    alpha = json.load(open(os.path.join(OUT, "c1_alpha.json")))["alpha"]
    s, q, v, params = c1_inputs()
    op = mhd_op(q, s.dx, s.dy, params)
    lin = ref_lin.FrozenLinearization(op, q.reshape(-1).copy())
    dt = adt / alpha
    shift = ref_leja.shift_and_scale(alpha * dt)
    ref_leja._coeff_cache.clear()
    before = op.calls
    t0 = time.perf_counter()
    res = ref_leja.apply_phi_leja(1, lambda x: ref_lin.jvp(lin, x), v, dt, shift, C1_TOL)
    sec = time.perf_counter() - t0
    th = blas_threads()
    os.makedirs(SCRATCH, exist_ok=True)
    np.save(os.path.join(SCRATCH, f"c1_p{adt:g}_t{th}.npy"), res.vector)
    meta = dict(adt=adt, alpha=alpha, dt=dt, q=shift.q, theta=shift.theta, tol=C1_TOL,
                iterations=res.iterations, converged=bool(res.converged),
                residual=res.residual, rhs_calls=op.calls - before,
                p_norm=float(np.linalg.norm(res.vector)), seconds=sec, blas_threads=th,
                cache_sizes=sorted(len(c) for c in ref_leja._coeff_cache.values()))
    with open(os.path.join(SCRATCH, f"c1_p{adt:g}_t{th}.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(json.dumps(meta), flush=True)


def c1_combine():
    """Primary = the 1-thread run; floor = its distance to the 8-thread run."""
    points = []
    arrays = {}
    for adt in C1_SWEEP:
        a = json.load(open(os.path.join(SCRATCH, f"c1_p{adt:g}_t1.json")))
        b = json.load(open(os.path.join(SCRATCH, f"c1_p{adt:g}_t8.json")))
        va = np.load(os.path.join(SCRATCH, f"c1_p{adt:g}_t1.npy"))
        vb = np.load(os.path.join(SCRATCH, f"c1_p{adt:g}_t8.npy"))
        floor = float(np.linalg.norm(va - vb) / np.linalg.norm(va))
        floor_sample = float(np.linalg.norm(va[::C1_STRIDE] - vb[::C1_STRIDE])
                             / np.linalg.norm(va[::C1_STRIDE]))
        pt = dict(a, floor_rel=floor, floor_rel_sample=floor_sample,
                  floor_iterations=b["iterations"], floor_converged=b["converged"],
                  floor_seconds=b["seconds"], p_sha256=sha(va))
        points.append(pt)
        arrays[f"p{adt:g}_sample"] = va[::C1_STRIDE]
        arrays[f"p{adt:g}_floor_sample"] = vb[::C1_STRIDE]
    meta = json.load(open(os.path.join(OUT, "c1_alpha.json")))
    meta.pop("generator", None)
    old = np.load(os.path.join(OUT, "c1_alpha.npz"))
    arrays["fu_sample"] = old["fu_sample"]
    save("c1", dict(meta, points=points, floor_method="reference with OPENBLAS_NUM_THREADS=1 "
                    "(primary) vs 8 (floor): another ddot summation order"), arrays)
    os.remove(os.path.join(OUT, "c1_alpha.npz"))
    os.remove(os.path.join(OUT, "c1_alpha.json"))


# ------------------------------------------------------ high-degree phi calls

def _fsum_norm(x):
    return math.sqrt(math.fsum(np.asarray(x, dtype=float).ravel() ** 2))


def degree_cases():
    """phi calls whose degree crosses the 64 -> 128 -> 256 coefficient-chunk
    boundaries (leja.py:119-130), plus a blow-up at the 256-chunk, each with a
    summation-order floor (the same call with a correctly rounded norm)."""
    cases = (("khm40", 40, "kh-modes", 3, ((1, 30.0), (1, 80.0), (1, 120.0), (4, 60.0))),
             ("harris48", 48, "harris", 0, ((1, 30.0), (1, 60.0), (1, 80.0))))
    arrays = {}
    metas = []
    for tag, n, kind, mseed, calls in cases:
        if kind == "harris":
            s = sc.harris_setup(n)
        else:
            s = sc.Setup(**{**sc.kh_setup(n).__dict__, "kind": "kh-modes",
                            "extra": {"mode_seed": mseed}})
        q = sc.initial_fields(s)
        params = MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa)
        op = mhd_op(q, s.dx, s.dy, params)
        lin = ref_lin.FrozenLinearization(op, q.reshape(-1).copy())
        est = ref_lin.estimate_alpha(lin, None, rng=np.random.default_rng(0))
        v = sc.unit_gaussian(q.size, 8)
        arrays[f"{tag}__u"] = q
        arrays[f"{tag}__v"] = v
        rec = dict(name=tag, nx=n, ny=n, dx=s.dx, dy=s.dy, mu=s.mu, eta=s.eta,
                   kappa=s.kappa, alpha=est.alpha, phi=[])
        for l, adt in calls:
            dt = adt / est.alpha
            shift = ref_leja.shift_and_scale(est.alpha * dt)
            ref_leja._coeff_cache.clear()
            before = op.calls
            res = ref_leja.apply_phi_leja(l, lambda x: ref_lin.jvp(lin, x), v, dt, shift, 1e-10)
            sizes = sorted(len(c) for c in ref_leja._coeff_cache.values())
            calls_used = op.calls - before
            # floor: the same call with correctly rounded norms everywhere
            saved = np.linalg.norm
            np.linalg.norm = lambda x, *a, **k: _fsum_norm(x)
            try:
                lin2 = ref_lin.FrozenLinearization(op, q.reshape(-1).copy())
                ref_leja._coeff_cache.clear()
                res2 = ref_leja.apply_phi_leja(l, lambda x: ref_lin.jvp(lin2, x), v, dt,
                                               shift, 1e-10)
            finally:
                np.linalg.norm = saved
            key = f"{tag}__phi_l{l}_a{adt:g}"
            arrays[key] = res.vector
            fl = (float(np.linalg.norm(res.vector - res2.vector) / np.linalg.norm(res.vector))
                  if res.converged and res2.converged else None)
            rec["phi"].append(dict(key=key, l=l, adt=adt, dt=dt, q=shift.q, theta=shift.theta,
                                   tol=1e-10, iterations=res.iterations,
                                   converged=bool(res.converged), residual=res.residual,
                                   rhs_calls=calls_used, cache_sizes=sizes,
                                   floor_iterations=res2.iterations, floor_rel=fl))
            print(json.dumps(rec["phi"][-1]), flush=True)
        metas.append(rec)
    save("degree", dict(cases=metas, floor_method="same call with math.fsum norms"), arrays)


# ------------------------------------------------------------ adaptive runs

def run_reference(setup, scheme, max_steps=1_000_000):
    q = sc.initial_fields(setup)
    params = MHDParams(mu=setup.mu, eta=setup.eta, kappa=setup.kappa)
    spec = Scenario(problem="custom", case_id=setup.name, nx=setup.nx, ny=setup.ny,
                    t_final=setup.t_final, x_min=setup.x_min, x_max=setup.x_max,
                    y_min=setup.y_min, y_max=setup.y_max, params=params, tol=setup.tol)
    state0 = StateGrid(setup.nx, setup.ny, setup.dx, setup.dy, q)
    u_hash = sha(q)
    saved = ref_harness.initialize
    ref_harness.initialize = lambda _spec: StateGrid(state0.nx, state0.ny, state0.dx,
                                                      state0.dy, state0.data.copy())
    ref_leja._coeff_cache.clear()
    try:
        t0 = time.perf_counter()
        rep = ref_harness.run(ref_harness.RunConfig(scenario=spec, scheme=scheme, method="leja",
                                                    tol=setup.tol, rng_seed=setup.seed,
                                                    max_steps=max_steps, wall_budget=1e9))
        wall = time.perf_counter() - t0
    finally:
        ref_harness.initialize = saved
    recs = [dict(t=s.t, dt=s.dt, error=s.error, rhs_calls=s.rhs_calls,
                 phi_iterations=s.phi_iterations, phi_applications=s.phi_applications,
                 accepted=s.accepted, cost=s.cost) for s in rep.steps]
    fin = rep.final_state.data
    meta = dict(name=setup.name, nx=setup.nx, ny=setup.ny, scheme=scheme.value,
                tol=setup.tol, t_final=setup.t_final, max_steps=max_steps,
                accepted=rep.accepted, rejected=rep.rejected, rhs_evals=rep.rhs_evals,
                phi_iterations=rep.phi_iterations,
                spectrum_rhs_evals=rep.spectrum_rhs_evals, status=rep.status,
                checksum=rep.checksum, max_divb=rep.max_divb, mass_drift=rep.mass_drift,
                t_reached=rep.t_reached, steps=recs, wall_seconds=wall,
                wall_seconds_per_step=wall / max(1, len(recs)), u0_sha256=u_hash,
                final_norm=float(np.linalg.norm(fin.reshape(-1))),
                final_field_norms=[float(np.linalg.norm(fin[f])) for f in range(8)],
                blas_threads=blas_threads())
    return meta, fin


def c2_full():
    """Config 2 (Harris 512^2, EXPRB54s4, tol 1e-6) to t_end = 10."""
    setup = sc.CONFIGS[2]()
    meta, fin = run_reference(setup, Scheme.EXPRB54S4)
    flat = fin.reshape(-1)
    save("c2", dict(meta, stride=C2_STRIDE), dict(final_sample=flat[::C2_STRIDE]))


def c3_first_steps():
    """Config 3 (KH 4096^2, EXPRB43, tol 1e-5): the first two step attempts."""
    setup = sc.CONFIGS[3]()
    meta, fin = run_reference(setup, Scheme.EXPRB43, max_steps=2)
    flat = fin.reshape(-1)
    save("c3", dict(meta, stride=C3_STRIDE), dict(final_sample=flat[::C3_STRIDE]))


# --------------------------------------------------------- config 4 strips

C4_STRIPS = ((0, 4), (2046, 2050), (4094, 4098), (8188, 8192))
C4_ADT = 10.0
C4_ALPHA = 2000.0       # nominal: one Leja term only needs (dt, q, theta)


def quantised_direction(n, seed):
    """A Gaussian direction rounded to multiples of 2^-8 with |k| <= 2^11, so
    that sum(w*w) is exact in ANY summation order (every square is an integer
    multiple of 2^-16 below 2^6, and 537 M of them stay below 2^53 units):
    ||w|| is then the same correctly rounded sqrt on the CPU and the GPU, and
    the FD step of the JVP / first Leja term is bitwise the reference's."""
    g = np.random.default_rng(seed).standard_normal(n)
    np.clip(g, -8.0, 8.0, out=g)
    g *= 256.0
    np.round(g, out=g)
    g *= 1.0 / 256.0
    return g


def c4_strips():
    """Config 4 (Harris 8192^2, eta 1e-3) strip checks: F(u), one JVP and the
    first Leja term (y_1 and p_1) on owned rows [j0, j1), computed by the
    reference on the padded rows [j0-2, j1+2) as a standalone periodic grid
    (the stencil footprint is 2 rows, mhd.py:143) with the GLOBAL norms."""
    setup = sc.CONFIGS[4]()
    n = setup.nx
    t0 = time.perf_counter()
    q = sc.initial_fields(setup)
    u = q.reshape(-1)
    unorm = float(np.linalg.norm(u))
    w = quantised_direction(u.size, 41).reshape(q.shape)
    wn2 = float(np.add.reduce((w * w).reshape(-1)))
    wnorm = float(np.linalg.norm(w.reshape(-1)))
    assert math.sqrt(wn2) == wnorm
    eps = (ref_lin._SQRT_EPS * max(1.0, unorm)) / max(wnorm, 1e-300)
    params = MHDParams(mu=setup.mu, eta=setup.eta, kappa=setup.kappa)
    dt = C4_ADT / C4_ALPHA
    shift = ref_leja.shift_and_scale(C4_ALPHA * dt)
    ref_leja._coeff_cache.clear()
    coeffs = ref_leja._newton_coeffs(1, shift.q, shift.theta, 64)
    xi = ref_leja.leja_points(500)
    arrays = {}
    strips = []
    for j0, j1 in C4_STRIPS:
        rows = np.arange(j0 - 2, j1 + 2) % n
        us = q[:, rows, :]
        ws = w[:, rows, :]
        g = StateGrid(n, rows.size, setup.dx, setup.dy, us.copy())
        fu = mhd_rhs(g, params).reshape(8, rows.size, n)
        # jvp (linearize.py:62-67) with the global eps: (F(u + eps*w) - F(u)) / eps
        x = us + (eps * ws)
        fx = mhd_rhs(StateGrid(n, rows.size, setup.dx, setup.dy, x), params)
        jw = ((fx.reshape(8, rows.size, n) - fu) / eps)
        # first Leja term (leja.py:121-140): y = v; w = J y; y = ((dt*w) - (q*y))/theta - xi0*y
        y1 = ((dt * jw) - (shift.q * ws)) / shift.theta - (xi[0] * ws)
        p1 = (coeffs[0] * ws) + (coeffs[1] * y1)
        own = slice(2, 2 + (j1 - j0))
        for name, a in (("f", fu), ("jw", jw), ("y1", y1), ("p1", p1)):
            arrays[f"r{j0}__{name}"] = np.ascontiguousarray(a[:, own, ::C4_COL_STRIDE])
        strips.append([j0, j1])
        print(f"strip {j0}-{j1} done {time.perf_counter() - t0:.0f}s", flush=True)
    save("c4", dict(n=n, strips=strips, col_stride=C4_COL_STRIDE, unorm=unorm, wnorm=wnorm,
                    eps=eps, w_seed=41, dt=dt, q=shift.q, theta=shift.theta,
                    c0=float(coeffs[0]), c1=float(coeffs[1]), xi0=float(xi[0]),
                    u_sha256=sha(q), w_sha256=sha(w), mu=setup.mu, eta=setup.eta,
                    kappa=setup.kappa, blas_threads=blas_threads(),
                    seconds=time.perf_counter() - t0), arrays)


def main():
    what = sys.argv[1]
    if what == "c1-alpha":
        c1_alpha()
    elif what == "c1-point":
        c1_point(sys.argv[2])
    elif what == "c1-combine":
        c1_combine()
    elif what == "degree":
        degree_cases()
    elif what == "c2":
        c2_full()
    elif what == "c3":
        c3_first_steps()
    elif what == "c4":
        c4_strips()
    else:
        raise SystemExit(f"unknown job {what!r}")


if __name__ == "__main__":
    main()
