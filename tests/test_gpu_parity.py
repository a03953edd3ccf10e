"""Parity of the sm_100a path with the reference (golden vectors) and the CPU oracle.

GPU tests (B200).  Bars (BASELINE.json north_star):
  * RHS: bit-identical values to the reference (np.array_equal).
  * JVP: bit-identical when ||w|| is exact in any summation order; otherwise
    <= 1e-10 relative L2 (the FD step amplifies ulp-level norm differences).
  * phi_l(dt J) v: <= 1e-10 relative L2, same iteration / RHS-call counts.
  * adaptive runs: same accepted/rejected sequence and RHS count, final
    state <= 1e-8 relative L2.
"""

import numpy as np
import pytest
import torch

import golden_io

pytestmark = pytest.mark.gpu

PHI_TOL = 1e-10
RUN_TOL = 1e-8


@pytest.fixture(scope="module")
def xb():
    import paper_2108_13622_b200 as pkg
    from paper_2108_13622_b200 import _lib
    _lib.load()
    return pkg


def rel(a, b):
    a = a.cpu().numpy() if torch.is_tensor(a) else np.asarray(a)
    b = b.cpu().numpy() if torch.is_tensor(b) else np.asarray(b)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb else 1.0)


def _params(xb, m):
    bcx = xb.Boundary.PERIODIC if m["periodic_x"] else xb.Boundary.REFLECTING
    bcy = xb.Boundary.PERIODIC if m["periodic_y"] else xb.Boundary.REFLECTING
    return xb.MHDParams(mu=m["mu"], eta=m["eta"], kappa=m["kappa"], gamma=m["gamma"],
                        mu0=m["mu0"], bc_x=bcx, bc_y=bcy)


RHS_CASES = [m for m in golden_io.meta()["rhs"] if m["name"] != "blowup"]


@pytest.mark.parametrize("case", RHS_CASES, ids=lambda m: m["name"])
def test_rhs_bitwise_vs_reference(xb, case):
    g = golden_io.arrays("rhs_cases")
    q = g[case["name"] + "__u"]
    params = _params(xb, case)
    ny, nx = q.shape[1:]
    # host-buffer path (reference-style StateGrid with a NumPy array)
    out = xb.mhd_rhs(xb.StateGrid(nx, ny, case["dx"], case["dy"], q.copy()), params)
    assert isinstance(out, np.ndarray)
    assert np.array_equal(out, g[case["name"] + "__f"])
    # device-resident path
    dev = xb.mhd_rhs(xb.StateGrid(nx, ny, case["dx"], case["dy"], torch.from_numpy(q).cuda()),
                     params)
    assert dev.is_cuda and np.array_equal(dev.cpu().numpy(), g[case["name"] + "__f"])


def test_rhs_blowup_reports_reference_cells(xb):
    m = {c["name"]: c for c in golden_io.meta()["rhs"]}["blowup"]
    q = golden_io.arrays("rhs_cases")["blowup__u"]
    params = xb.MHDParams(mu=m["mu"], eta=m["eta"], kappa=m["kappa"])
    with pytest.raises(xb.RhsBlowupError) as err:
        xb.mhd_rhs(xb.StateGrid(16, 12, m["dx"], m["dy"], q.copy()), params)
    assert [list(c) for c in err.value.cells] == m["cells"]
    assert str(err.value) == m["message"]


def test_rhs_ieee_division_build_agrees(xb, monkeypatch):
    """The Markstein constant-divisor path equals true IEEE division on real states."""
    from paper_2108_13622_b200 import _lib, scenarios as sc
    for setup in (sc.harris_setup(96), sc.kh_setup(96)):
        q = torch.from_numpy(sc.initial_fields(setup)).cuda().reshape(-1)
        outs = []
        for ieee in ("0", "1"):
            monkeypatch.setenv("XMHD_DIV_IEEE", ieee)
            ctx = _lib.Context(setup.nx, setup.ny, setup.dx, setup.dy, setup.mu, setup.eta,
                               setup.kappa, setup.gamma, setup.mu0, 0, 0)
            f = torch.empty_like(q)
            assert _lib.load().xmhd_rhs(ctx.bind_stream(), _lib.ptr(q), _lib.ptr(f), None) == 0
            outs.append(f.cpu().numpy())
        assert np.array_equal(outs[0], outs[1])


def _lin(xb, g, case, tag):
    q = g[tag + "__u"]
    ny, nx = q.shape[1:]
    st = xb.StateGrid(nx, ny, case["dx"], case["dy"], torch.from_numpy(q).cuda())
    params = xb.MHDParams(mu=case["mu"], eta=case["eta"], kappa=case["kappa"])
    op = xb.RhsOperator(xb.MhdRhs(st, params))
    return op, xb.FrozenLinearization(op, st.flat())


LEJA_CASES = golden_io.meta()["leja"]


@pytest.mark.parametrize("case", LEJA_CASES, ids=lambda m: m["name"])
def test_jvp_vs_reference(xb, case):
    g = golden_io.arrays("leja_cases")
    tag = case["name"]
    op, lin = _lin(xb, g, case, tag)
    assert np.array_equal(lin.base_rhs.cpu().numpy(), g[tag + "__fu"])
    calls = op.calls
    jw = xb.jvp(lin, torch.from_numpy(g[tag + "__w"]).cuda())
    assert op.calls == calls + 1
    assert rel(jw, g[tag + "__jw"]) <= PHI_TOL


def test_jvp_bitwise_with_exact_norm(xb):
    """With ||w|| exact in any order, the fused JVP equals the oracle bit for bit."""
    from oracle import leja_np as olj, mhd_np
    from paper_2108_13622_b200 import scenarios as sc
    s = sc.kh_setup(64)
    q = sc.initial_fields(s)
    w = np.random.default_rng(4).integers(-8, 9, size=q.size).astype(float) * 2.0 ** -5
    st = xb.StateGrid(s.nx, s.ny, s.dx, s.dy, torch.from_numpy(q).cuda())
    params = xb.MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa)
    lin = xb.FrozenLinearization(xb.RhsOperator(xb.MhdRhs(st, params)), st.flat())
    # ||u|| also enters eps; give both sides the same value
    f = lambda flat: mhd_np.rhs(flat.reshape(q.shape), s.dx, s.dy, s.mu, s.eta, s.kappa)
    olin = olj.Frozen(olj.CountedRhs(f), q.reshape(-1))
    olin.unorm = lin._base_norm
    jw = xb.jvp(lin, torch.from_numpy(w).cuda()).cpu().numpy()
    assert np.array_equal(jw, olj.fd_jvp(olin, w))


def test_jvp_zero_vector_costs_nothing(xb):
    from paper_2108_13622_b200 import scenarios as sc
    s = sc.kh_setup(16)
    st = xb.StateGrid(s.nx, s.ny, s.dx, s.dy, torch.from_numpy(sc.initial_fields(s)).cuda())
    op = xb.RhsOperator(xb.MhdRhs(st, xb.MHDParams(1e-3, 1e-3, 1e-3)))
    lin = xb.FrozenLinearization(op, st.flat())
    calls = op.calls
    out = xb.jvp(lin, torch.zeros_like(st.flat()))
    assert op.calls == calls and torch.count_nonzero(out) == 0


@pytest.mark.parametrize("case", LEJA_CASES, ids=lambda m: m["name"])
def test_power_iteration_vs_reference(xb, case):
    g = golden_io.arrays("leja_cases")
    op, lin = _lin(xb, g, case, case["name"])
    calls = op.calls
    est = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0))
    assert op.calls - calls == case["power_calls"]
    assert abs(est.alpha - case["alpha"]) <= 1e-10 * case["alpha"]
    assert rel(est.vector, g[case["name"] + "__power_vec"]) <= 1e-9


PHI_CASES = [(m, p) for m in LEJA_CASES for p in m["phi"]]


@pytest.mark.parametrize("case,phi", PHI_CASES, ids=lambda x: x.get("key", ""))
def test_phi_leja_vs_reference(xb, case, phi):
    from paper_2108_13622_b200 import leja
    g = golden_io.arrays("leja_cases")
    op, lin = _lin(xb, g, case, case["name"])
    leja._coeff_cache.clear()
    v = torch.from_numpy(g[case["name"] + "__v"]).cuda()
    calls = op.calls
    res = xb.apply_phi_leja(phi["l"], xb.JacobianAction(lin), v, phi["dt"],
                            xb.ShiftScale(phi["q"], phi["theta"]), phi["tol"])
    assert res.iterations == phi["iterations"]
    assert res.converged == phi["converged"]
    assert op.calls - calls == phi["rhs_calls"]
    assert rel(res.vector, g[phi["key"]]) <= PHI_TOL


STEP_CASES = golden_io.meta()["step"]


@pytest.mark.parametrize("case", STEP_CASES, ids=lambda m: m["name"])
def test_single_step_vs_reference(xb, case):
    from paper_2108_13622_b200 import leja
    g = golden_io.arrays("step_cases")
    op, lin = _lin(xb, g, case, case["name"])
    est = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0))
    leja._coeff_cache.clear()
    before = op.calls
    res = xb.step(xb.Scheme(case["scheme"]), op, lin.base_state, case["dt"], alpha=est,
                  tol=case["tol"], lin=lin)
    assert res.converged == case["converged"]
    assert res.rhs_calls == case["rhs_calls"] == op.calls - before
    assert res.phi_iterations == case["phi_iterations"]
    assert res.phi_applications == case["phi_applications"]
    assert abs(res.error_estimate - case["error"]) <= 1e-6 * case["error"]
    assert rel(res.new_state, g[case["name"] + "__new"]) <= PHI_TOL


RUN_CASES = golden_io.meta()["run"]


@pytest.mark.parametrize("case", RUN_CASES, ids=lambda m: m["name"])
def test_adaptive_run_vs_reference(xb, case):
    from paper_2108_13622_b200 import leja, scenarios as sc
    if case["name"] == "C0":
        setup = sc.kh_setup(128)
    elif case["name"].startswith("C2"):
        setup = sc.harris_setup(case["nx"], t_final=case["t_final"])
    else:
        setup = sc.kh_setup(case["nx"], t_final=case["t_final"])
    leja._coeff_cache.clear()
    rep = xb.run(xb.RunConfig(scenario=setup, scheme=xb.Scheme(case["scheme"]),
                              tol=case["tol"], rng_seed=setup.seed))
    assert rep.status == case["status"]
    assert (rep.accepted, rep.rejected) == (case["accepted"], case["rejected"])
    assert [s.accepted for s in rep.steps] == [s["accepted"] for s in case["steps"]]
    assert [s.rhs_calls for s in rep.steps] == [s["rhs_calls"] for s in case["steps"]]
    assert rep.rhs_evals == case["rhs_evals"]
    assert rep.phi_iterations == case["phi_iterations"]
    assert rep.spectrum_rhs_evals == case["spectrum_rhs_evals"]
    final = golden_io.arrays("run_cases")[case["name"] + "__final"]
    assert rel(rep.final_state.data, final) <= RUN_TOL
    assert abs(rep.t_reached - case["t_reached"]) <= 1e-12


def test_run_is_bit_deterministic(xb):
    from paper_2108_13622_b200 import scenarios as sc
    setup = sc.kh_setup(32, t_final=0.05)
    a = xb.run(xb.RunConfig(scenario=setup))
    b = xb.run(xb.RunConfig(scenario=setup))
    assert a.checksum == b.checksum and a.rhs_evals == b.rhs_evals
    assert [s.dt for s in a.steps] == [s.dt for s in b.steps]


def test_diagnostics_vs_oracle(xb):
    from oracle import mhd_np
    from paper_2108_13622_b200 import harness, scenarios as sc
    s = sc.harris_setup(64)
    q = sc.initial_fields(s)
    st = xb.StateGrid(s.nx, s.ny, s.dx, s.dy, q.copy())
    params = xb.MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa)
    assert np.array_equal(xb.discrete_div_b(st, params), mhd_np.div_b(q, s.dx, s.dy))
    assert harness.initial_dt(st, params) == mhd_np.initial_dt(q, s.dx, s.dy)
    tot = xb.conserved_totals(st)
    for k, v in mhd_np.totals(q, s.dx, s.dy).items():
        assert tot[k] == pytest.approx(v, rel=1e-12, abs=1e-12)


def test_generic_matvec_diagonal_example(xb):
    a = np.diag([-1.0, -10.0])
    res = xb.apply_phi_leja(1, lambda w: a @ w, np.ones(2), 0.1, xb.shift_and_scale(10.0),
                            1e-10)
    assert res.converged
    expect = np.array([xb.phi_scalar(1, -0.1), xb.phi_scalar(1, -1.0)])
    assert np.allclose(res.vector, expect, rtol=1e-9)


def test_generic_matvec_matches_oracle_bitwise(xb):
    """Generic matvec path: vector algebra on the device equals NumPy's."""
    from oracle import leja_np as olj
    rng = np.random.default_rng(5)
    eig = rng.uniform(-20.0, 0.0, 24)
    qm, _ = np.linalg.qr(rng.standard_normal((24, 24)))
    a = qm @ np.diag(eig) @ qm.T
    v = rng.integers(-4, 5, 24).astype(float)
    sh = xb.shift_and_scale(25.0)
    calls = [0]

    def mv(w):
        calls[0] += 1
        return a @ w
    res = xb.apply_phi_leja(1, mv, v, 1.0, sh, 1e-10)
    ref = olj.phi_leja(1, lambda w: a @ w, v, 1.0, sh.q, sh.theta, 1e-10, olj.CoeffCache())
    assert res.converged and res.iterations == ref.iterations == calls[0]
    assert rel(res.vector, ref.vector) <= 1e-13


def test_leja_nonconvergence_is_a_flag(xb):
    a = np.diag([-1000.0])
    res = xb.apply_phi_leja(1, lambda w: a @ w, np.ones(1), 1.0, xb.shift_and_scale(1.0),
                            1e-10)
    assert not res.converged and res.iterations <= 500


def test_rhs_large_grid_vs_oracle(xb):
    """2048^2 RHS equals the oracle on periodic strips (F is local: rows j0-2..j1+2)."""
    from oracle import mhd_np
    from paper_2108_13622_b200 import scenarios as sc
    s = sc.CONFIGS[1]()
    q = sc.initial_fields(s)
    f = xb.mhd_rhs(xb.StateGrid(s.nx, s.ny, s.dx, s.dy, torch.from_numpy(q).cuda()),
                   xb.MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa)).cpu().numpy()
    f = f.reshape(q.shape)
    for j0 in (0, 777, 2040):
        rows = [(j0 + k) % s.ny for k in range(-2, 10)]
        strip = q[:, rows, :]
        ref = mhd_np.rhs(strip, s.dx, s.dy, s.mu, s.eta, s.kappa).reshape(strip.shape)
        got = f[:, [(j0 + k) % s.ny for k in range(0, 8)], :]
        assert np.array_equal(got, ref[:, 2:10, :])


BC_CASES = golden_io.meta()["leja_bc"]


@pytest.mark.parametrize("case", BC_CASES, ids=lambda m: m["name"])
def test_leja_boundaries_vs_reference(xb, case):
    """Reflecting walls in x and/or y, mu0 != 1, gamma != 5/3, ideal MHD and
    non-power-of-two spacings (Markstein division kinds) through the fused
    JVP, the power iteration and the fused Leja loop."""
    from paper_2108_13622_b200 import leja
    g = golden_io.arrays("leja_bc_cases")
    tag = case["name"]
    q = g[tag + "__u"]
    ny, nx = q.shape[1:]
    st = xb.StateGrid(nx, ny, case["dx"], case["dy"], torch.from_numpy(q).cuda())
    op = xb.RhsOperator(xb.MhdRhs(st, _params(xb, case)))
    lin = xb.FrozenLinearization(op, st.flat())
    assert np.array_equal(lin.base_rhs.cpu().numpy(), g[tag + "__fu"])
    jw = xb.jvp(lin, torch.from_numpy(g[tag + "__w"]).cuda())
    assert rel(jw, g[tag + "__jw"]) <= PHI_TOL
    calls = op.calls
    est = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0))
    assert op.calls - calls == case["power_calls"]
    assert abs(est.alpha - case["alpha"]) <= 1e-10 * case["alpha"]
    v = torch.from_numpy(g[tag + "__v"]).cuda()
    for p in case["phi"]:
        leja._coeff_cache.clear()
        calls = op.calls
        res = xb.apply_phi_leja(p["l"], xb.JacobianAction(lin), v, p["dt"],
                                xb.ShiftScale(p["q"], p["theta"]), p["tol"])
        assert (res.iterations, res.converged) == (p["iterations"], p["converged"]), p["key"]
        assert op.calls - calls == p["rhs_calls"]
        assert rel(res.vector, g[p["key"]]) <= PHI_TOL, p["key"]
