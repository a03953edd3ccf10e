"""y-strip decomposition on the GPU.

Only one GPU is available to the tests, so multi-rank runs emulate ranks with
host threads on that GPU (tests/strip_emul.py); the real transport is
torch.distributed (NCCL), whose orchestration is covered on CPU with gloo in
tests/test_strips_cpu.py.  Bars:
  * strip RHS / JVP (BC_HALO kernels) == the single-domain kernels bit for bit;
  * phi_l on P strips == single domain to 1e-12 (norms summed per strip);
  * adaptive runs on P strips: same step sequence and RHS counts as the
    reference, final state <= 1e-8.
"""

import numpy as np
import pytest
import torch

import golden_io
from strip_emul import run_ranks

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = a.cpu().numpy() if torch.is_tensor(a) else np.asarray(a)
    b = b.cpu().numpy() if torch.is_tensor(b) else np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _problem(n=48, refl=False):
    import paper_2108_13622_b200 as xb
    from paper_2108_13622_b200 import scenarios as sc
    s = sc.Setup(**{**sc.kh_setup(n).__dict__, "kind": "kh-modes", "ny": n + 6,
                    "extra": {"mode_seed": 4}})
    q = sc.initial_fields(s)
    bcy = xb.Boundary.REFLECTING if refl else xb.Boundary.PERIODIC
    params = xb.MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa, bc_y=bcy)
    return s, q, params


@pytest.mark.parametrize("refl", [False, True])
@pytest.mark.parametrize("nranks", [1, 2, 3])
def test_strip_rhs_and_jvp_bitwise(refl, nranks):
    import paper_2108_13622_b200 as xb
    from paper_2108_13622_b200 import strips
    s, q, params = _problem(refl=refl)
    geo = xb.StateGrid(s.nx, s.ny, s.dx, s.dy, torch.from_numpy(q).cuda())
    f_ref = xb.mhd_rhs(geo, params).cpu().numpy().reshape(q.shape)
    w = np.random.default_rng(3).standard_normal(q.shape)
    lin = xb.FrozenLinearization(xb.RhsOperator(xb.MhdRhs(geo, params)), geo.flat())
    eps = 1e-7
    from paper_2108_13622_b200 import _lib
    jv_ref = torch.empty_like(lin.base_state)
    rc = _lib.load().xmhd_jvp_eps(lin.mhd.ctx.bind_stream(), _lib.ptr(lin.base_state),
                                  _lib.ptr(lin.base_rhs), _lib.ptr(torch.from_numpy(w).cuda()
                                                                   .reshape(-1)),
                                  eps, _lib.ptr(jv_ref), None)
    assert rc == 0
    jv_ref = jv_ref.cpu().numpy().reshape(q.shape)

    def rank(comm):
        mhd = strips.StripMhd(xb.StateGrid(s.nx, s.ny, s.dx, s.dy, None), params, comm)
        lay = mhd.layout
        u = torch.from_numpy(np.ascontiguousarray(lay.local_rows(q))).cuda().reshape(-1)
        f = mhd(u)
        wl = torch.from_numpy(np.ascontiguousarray(lay.local_rows(w))).cuda().reshape(-1)
        fu_l = torch.from_numpy(np.ascontiguousarray(lay.local_rows(f_ref))).cuda().reshape(-1)
        jv, bad = mhd.jvp(u, fu_l, wl, eps)
        assert not bad
        return lay.y0, lay.ny, f.cpu().numpy(), jv.cpu().numpy()

    for y0, ny, f, jv in run_ranks(nranks, rank):
        assert np.array_equal(f.reshape(8, ny, s.nx), f_ref[:, y0:y0 + ny])
        assert np.array_equal(jv.reshape(8, ny, s.nx), jv_ref[:, y0:y0 + ny])


@pytest.mark.parametrize("nranks", [1, 2, 3])
def test_strip_phi_matches_single_domain(nranks):
    import paper_2108_13622_b200 as xb
    from paper_2108_13622_b200 import leja, scenarios as sc, strips
    s, q, params = _problem(64)
    v = sc.unit_gaussian(q.size, 9).reshape(q.shape)
    geo = xb.StateGrid(s.nx, s.ny, s.dx, s.dy, torch.from_numpy(q).cuda())
    op = xb.RhsOperator(xb.MhdRhs(geo, params))
    lin = xb.FrozenLinearization(op, geo.flat())
    alpha = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0)).alpha
    refs = {}
    for adt in (2.0, 40.0):
        leja._coeff_cache.clear()
        sh = xb.shift_and_scale(adt)
        refs[adt] = xb.apply_phi_leja(1, xb.JacobianAction(lin),
                                      torch.from_numpy(v).cuda().reshape(-1), adt / alpha, sh,
                                      1e-10)

    def rank(comm):
        mhd = strips.StripMhd(xb.StateGrid(s.nx, s.ny, s.dx, s.dy, None), params, comm)
        prev = xb.linearize._ops.set_reducer(strips.Reducer(comm, torch.device("cuda")))
        try:
            lay = mhd.layout
            u = torch.from_numpy(np.ascontiguousarray(lay.local_rows(q))).cuda().reshape(-1)
            sop = xb.RhsOperator(mhd)
            slin = xb.FrozenLinearization(sop, u)
            vl = torch.from_numpy(np.ascontiguousarray(lay.local_rows(v))).cuda().reshape(-1)
            out = {}
            for adt in (2.0, 40.0):
                res = xb.apply_phi_leja(1, xb.JacobianAction(slin), vl, adt / alpha,
                                        xb.shift_and_scale(adt), 1e-10)
                out[adt] = (res.iterations, res.converged, res.vector.cpu().numpy(), sop.calls)
            return lay.y0, lay.ny, out
        finally:
            xb.linearize._ops.set_reducer(prev)

    results = run_ranks(nranks, rank)
    for adt, ref in refs.items():
        full = np.concatenate([r[2][adt][2].reshape(8, r[1], s.nx) for r in results], axis=1)
        for r in results:
            assert r[2][adt][0] == ref.iterations and r[2][adt][1] == ref.converged
        # strip-wise norm sums differ in the last ulps; the FD step amplifies it
        # with the degree (the CPU-vs-CPU floor of SURVEY §8(c))
        # (measured: ~1e-14 at alpha*dt=2; ~5e-9 at alpha*dt=40, degree 106)
        assert rel(full.reshape(-1), ref.vector) <= (1e-12 if adt <= 10 else 1e-7)


@pytest.mark.parametrize("nranks", [2, 3])
def test_strip_adaptive_run_vs_reference(nranks):
    import paper_2108_13622_b200 as xb
    from paper_2108_13622_b200 import scenarios as sc
    case = {c["name"]: c for c in golden_io.meta()["run"]}["C0_32_t0.2"]
    setup = sc.kh_setup(case["nx"], t_final=case["t_final"])

    def rank(comm):
        return xb.run(xb.RunConfig(scenario=setup, scheme=xb.Scheme(case["scheme"]),
                                   tol=case["tol"]), comm=comm)

    reps = run_ranks(nranks, rank)
    rep = reps[0]
    assert rep.status == case["status"]
    assert [s.rhs_calls for s in rep.steps] == [s["rhs_calls"] for s in case["steps"]]
    assert rep.rhs_evals == case["rhs_evals"]
    for other in reps[1:]:
        assert [s.dt for s in other.steps] == [s.dt for s in rep.steps]
        assert other.final_state is None
    final = golden_io.arrays("run_cases")[case["name"] + "__final"]
    assert rel(rep.final_state.data, final) <= 1e-8
    assert abs(rep.max_divb - case["max_divb"]) <= 1e-12 + 1e-6 * case["max_divb"]


@pytest.mark.parametrize("nranks", [2, 3])
def test_strip_krylov_matches_single_domain(nranks):
    """The Krylov arm on y-strips: every MGS coefficient reduced over the ranks."""
    import paper_2108_13622_b200 as xb
    from paper_2108_13622_b200 import scenarios as sc, strips
    s, q, params = _problem(48)
    v = sc.unit_gaussian(q.size, 9).reshape(q.shape)
    geo = xb.StateGrid(s.nx, s.ny, s.dx, s.dy, torch.from_numpy(q).cuda())
    lin = xb.FrozenLinearization(xb.RhsOperator(xb.MhdRhs(geo, params)), geo.flat())
    alpha = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0)).alpha
    dt = 5.0 / alpha
    ref = xb.apply_phi_krylov(1, xb.JacobianAction(lin), torch.from_numpy(v).cuda().reshape(-1),
                              dt, 1e-10)

    def rank(comm):
        mhd = strips.StripMhd(xb.StateGrid(s.nx, s.ny, s.dx, s.dy, None), params, comm)
        prev = xb.linearize._ops.set_reducer(strips.Reducer(comm, torch.device("cuda")))
        try:
            lay = mhd.layout
            u = torch.from_numpy(np.ascontiguousarray(lay.local_rows(q))).cuda().reshape(-1)
            slin = xb.FrozenLinearization(xb.RhsOperator(mhd), u)
            vl = torch.from_numpy(np.ascontiguousarray(lay.local_rows(v))).cuda().reshape(-1)
            res = xb.apply_phi_krylov(1, xb.JacobianAction(slin), vl, dt, 1e-10)
            return lay.y0, lay.ny, res.iterations, res.converged, res.vector.cpu().numpy()
        finally:
            xb.linearize._ops.set_reducer(prev)

    results = run_ranks(nranks, rank)
    full = np.concatenate([r[4].reshape(8, r[1], s.nx) for r in results], axis=1)
    for r in results:
        assert (r[2], r[3]) == (ref.iterations, ref.converged)
    assert rel(full.reshape(-1), ref.vector) <= 1e-11
