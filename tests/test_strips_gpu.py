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


@pytest.mark.parametrize("nranks,refl", [(2, False), (3, False), (3, True)])
def test_strip_peer_transport_emulated(nranks, refl):
    """The peer-memory Leja loop (boundary rows pushed into the neighbours'
    ghost rows and the sums all-reduced through peer boards, all inside the
    fused kernel), with the ranks emulated in ONE cooperative launch per term on
    this GPU: bit-identical to the NCCL-style strip loop (same sums in the same
    rank order), same iteration counts."""
    import ctypes
    import paper_2108_13622_b200 as xb
    from paper_2108_13622_b200 import _lib, leja, scenarios as sc, strips
    s, q, params = _problem(48, refl=refl)
    v = sc.unit_gaussian(q.size, 9).reshape(q.shape)
    geo = xb.StateGrid(s.nx, s.ny, s.dx, s.dy, torch.from_numpy(q).cuda())
    lin = xb.FrozenLinearization(xb.RhsOperator(xb.MhdRhs(geo, params)), geo.flat())
    alpha = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0)).alpha
    cases = [(1, 2.0), (2, 30.0)]

    def rank(comm):
        mhd = strips.StripMhd(xb.StateGrid(s.nx, s.ny, s.dx, s.dy, None), params, comm)
        prev = xb.linearize._ops.set_reducer(strips.Reducer(comm, torch.device("cuda")))
        try:
            lay = mhd.layout
            u = torch.from_numpy(np.ascontiguousarray(lay.local_rows(q))).cuda().reshape(-1)
            slin = xb.FrozenLinearization(xb.RhsOperator(mhd), u)
            vl = torch.from_numpy(np.ascontiguousarray(lay.local_rows(v))).cuda().reshape(-1)
            out = []
            for l, adt in cases:
                res = xb.apply_phi_leja(l, xb.JacobianAction(slin), vl, adt / alpha,
                                        xb.shift_and_scale(adt), 1e-10)
                out.append((res.iterations, res.converged, res.vector.cpu().numpy()))
            mhd.exchange(slin.base_state, mhd.state_halo)
            mhd._set_halo(mhd.state_halo, mhd.dir_halo)
            torch.cuda.current_stream().synchronize()
            return mhd, slin, vl, out
        finally:
            xb.linearize._ops.set_reducer(prev)

    results = run_ranks(nranks, rank)
    lib = _lib.load()
    P = nranks
    ctxs = (ctypes.c_void_p * P)(*[r[0].ctx.bind_stream().value for r in results])
    for r in results:
        buf = (ctypes.c_char * 64)()
        _lib.check(lib.xmhd_p2p_alloc(r[0].ctx.h, buf), "xmhd_p2p_alloc")
    _lib.check(lib.xmhd_p2p_connect_local(ctxs, P, int(not refl)), "xmhd_p2p_connect_local")
    ptrs = lambda ts: (ctypes.c_void_p * P)(*[t.data_ptr() for t in ts])
    u_p = ptrs([r[1].base_state for r in results])
    f_p = ptrs([r[1].base_rhs for r in results])
    v_p = ptrs([r[2] for r in results])
    unorm = float(results[0][1]._base_norm)
    xi = np.ascontiguousarray(leja.leja_points(500))
    dp = ctypes.POINTER(ctypes.c_double)
    for k, (l, adt) in enumerate(cases):
        sh = xb.shift_and_scale(adt)
        chunk = 64
        coeffs = np.ascontiguousarray(leja._newton_coeffs(l, sh.q, sh.theta, chunk))
        rc = lib.xmhd_leja_p2p_emul_start(ctxs, P, u_p, f_p, unorm, v_p, adt / alpha, sh.q,
                                          sh.theta, 1e-10, xi.ctypes.data_as(dp),
                                          coeffs.ctypes.data_as(dp), coeffs.size)
        _lib.check(rc, "xmhd_leja_p2p_emul_start")
        st = _lib.LejaState()
        _lib.check(lib.xmhd_leja_p2p_emul_run(ctxs, P, ctypes.byref(st)), "emul_run")
        while st.status == _lib.LEJA_NEED_COEFFS:
            chunk, coeffs = leja._grow(l, sh.q, sh.theta, chunk, coeffs, st.m)
            coeffs = np.ascontiguousarray(coeffs)
            for r in results:
                _lib.check(lib.xmhd_leja_set_coeffs(r[0].ctx.h, coeffs.ctypes.data_as(dp),
                                                    coeffs.size), "set_coeffs")
            _lib.check(lib.xmhd_leja_p2p_emul_run(ctxs, P, ctypes.byref(st)), "emul_run")
        assert st.status == _lib.LEJA_CONVERGED
        for r in results:
            its, conv, ref_vec = r[3][k]
            assert st.iterations == its and conv
            p = torch.empty_like(r[2])
            _lib.check(lib.xmhd_leja_result(r[0].ctx.h, _lib.ptr(p)), "xmhd_leja_result")
            assert np.array_equal(p.cpu().numpy(), ref_vec), (k, r[0].layout.y0)


def test_peer_transport_setup_errors():
    import ctypes
    import paper_2108_13622_b200 as xb
    from paper_2108_13622_b200 import _lib
    lib = _lib.load()
    c = _lib.Context(16, 8, 0.1, 0.1, 0.01, 0.01, 0.01, 5.0 / 3.0, 1.0, _lib.BC_PERIODIC,
                     _lib.BC_PERIODIC)
    buf = (ctypes.c_char * 64)()
    assert lib.xmhd_p2p_alloc(c.h, buf) == 2            # not a y-strip context
    s = _lib.Context(16, 8, 0.1, 0.1, 0.01, 0.01, 0.01, 5.0 / 3.0, 1.0, _lib.BC_PERIODIC,
                     _lib.BC_HALO)
    st = _lib.LejaState()
    assert lib.xmhd_leja_p2p_run(s.h, ctypes.byref(st)) == 2   # not connected
    assert lib.xmhd_p2p_alloc(s.h, buf) == 0
    handles = (ctypes.c_char * 128)()
    assert lib.xmhd_p2p_connect(s.h, 0, 1, handles, 1) == 2    # one rank: no peers
    assert lib.xmhd_p2p_connect(s.h, 2, 2, handles, 1) == 2    # rank out of range
