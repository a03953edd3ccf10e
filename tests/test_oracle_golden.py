"""Pin the CPU oracle to the golden vectors produced by the reference itself.

CPU-only.  The oracle (``oracle/``) must reproduce the reference bit for bit
where the reference's arithmetic is deterministic NumPy ufuncs (RHS, JVP,
divided differences, Leja points), and to the BLAS-norm floor elsewhere.
"""

import numpy as np
import pytest

import golden_io
from oracle import leja_np as lj
from oracle import mhd_np
from oracle import steppers_np as st


def _rhs_meta():
    return {m["name"]: m for m in golden_io.meta()["rhs"]}


@pytest.mark.parametrize("name", [m["name"] for m in golden_io.meta()["rhs"]
                                  if m["name"] != "blowup"])
def test_oracle_rhs_bitwise(name):
    m = _rhs_meta()[name]
    g = golden_io.arrays("rhs_cases")
    out = mhd_np.rhs(g[f"{name}__u"], m["dx"], m["dy"], m["mu"], m["eta"], m["kappa"],
                     m["gamma"], m["mu0"], m["periodic_x"], m["periodic_y"])
    assert np.array_equal(out, g[f"{name}__f"])


def test_oracle_rhs_blowup_cells():
    m = _rhs_meta()["blowup"]
    g = golden_io.arrays("rhs_cases")
    with pytest.raises(mhd_np.NonFiniteRhs) as err:
        mhd_np.rhs(g["blowup__u"], m["dx"], m["dy"], m["mu"], m["eta"], m["kappa"])
    assert [list(c) for c in err.value.cells] == m["cells"]
    assert str(err.value) == m["message"]


def test_oracle_leja_points_bitwise():
    g = golden_io.arrays("coeff_cases")
    assert np.array_equal(lj.leja_points(500), g["leja_points"])


def test_oracle_coefficients_bitwise():
    g = golden_io.arrays("coeff_cases")
    for m in golden_io.meta()["coeff"]:
        cache = lj.CoeffCache()
        c = cache.get(m["l"], m["q"], m["theta"], m["count"])
        assert np.array_equal(c, g[m["key"]]), m["key"]
    nodes = lj.leja_points(64)
    for l in (0, 1, 3):
        assert np.array_equal(lj.phi_divdiff(l, nodes), g[f"divdiff_l{l}"])


def _lin(g, m, tag):
    q = g[f"{tag}__u"]

    def f(flat):
        return mhd_np.rhs(flat.reshape(q.shape), m["dx"], m["dy"], m["mu"], m["eta"],
                          m["kappa"])
    op = lj.CountedRhs(f)
    return op, lj.Frozen(op, q.reshape(-1).copy())


@pytest.mark.parametrize("case", golden_io.meta()["leja"], ids=lambda m: m["name"])
def test_oracle_jvp_power_and_phi(case):
    g = golden_io.arrays("leja_cases")
    tag = case["name"]
    op, lin = _lin(g, case, tag)
    assert np.array_equal(lin.fu, g[f"{tag}__fu"])
    assert np.array_equal(lj.fd_jvp(lin, g[f"{tag}__w"]), g[f"{tag}__jw"])
    calls = op.calls
    est = lj.power_alpha(lin, None, rng=np.random.default_rng(0))
    assert op.calls - calls == case["power_calls"]
    assert est.alpha == case["alpha"]
    assert np.array_equal(est.vector, g[f"{tag}__power_vec"])
    v = g[f"{tag}__v"]
    for p in case["phi"]:
        calls = op.calls
        res = lj.phi_leja(p["l"], lambda x: lj.fd_jvp(lin, x), v, p["dt"], p["q"],
                          p["theta"], p["tol"], lj.CoeffCache())
        assert res.iterations == p["iterations"]
        assert res.converged == p["converged"]
        assert op.calls - calls == p["rhs_calls"]
        assert np.array_equal(res.vector, g[p["key"]]), p["key"]
        assert res.residual == p["residual"]


@pytest.mark.parametrize("case", golden_io.meta()["step"], ids=lambda m: m["name"])
def test_oracle_single_step(case):
    g = golden_io.arrays("step_cases")
    tag = case["name"]
    op, lin = _lin(g, case, tag)
    est = lj.power_alpha(lin, None, rng=np.random.default_rng(0))
    assert est.alpha == case["alpha"]
    before = op.calls
    res = st.one_step(case["scheme"], op, lin.u, case["dt"], est, case["tol"], lin,
                      lj.CoeffCache())
    assert res.converged == case["converged"]
    assert res.rhs_calls == case["rhs_calls"] == op.calls - before
    assert res.phi_iterations == case["phi_iterations"]
    assert res.phi_applications == case["phi_applications"]
    assert res.error_estimate == case["error"]
    assert np.array_equal(res.new_state, g[f"{tag}__new"])


def test_oracle_controllers_worked_examples():
    # SPEC worked examples as exercised by the reference's acceptance criterion 5
    assert abs(st.cost_next(0.1, 0.05, 100.0, 100.0) - 0.1 * 1.37412002) <= 1e-12
    assert abs(st.cost_next(0.1, 0.05, 200.0, 100.0) - 0.1 * 0.64446017) <= 1e-12
    assert st.trad_next(0.1, 0.0, 1e-4, 3) == 0.2
    assert st.trad_next(0.1, 1e9, 1e-4, 3) == 0.05


@pytest.mark.parametrize("case", golden_io.meta()["run"], ids=lambda m: m["name"])
def test_oracle_adaptive_run(case):
    from paper_2108_13622_b200 import scenarios as sc
    if case["name"] == "C0":
        setup = sc.kh_setup(128)
    elif case["name"].startswith("C2"):
        setup = sc.harris_setup(case["nx"], t_final=case["t_final"])
    else:
        setup = sc.kh_setup(case["nx"], t_final=case["t_final"])
    q = sc.initial_fields(setup)
    rep = st.run(q, setup.dx, setup.dy, setup.mu, setup.eta, setup.kappa,
                 case["scheme"], case["tol"], case["t_final"], cache=lj.CoeffCache())
    assert rep.status == case["status"]
    assert (rep.accepted, rep.rejected) == (case["accepted"], case["rejected"])
    assert rep.rhs_evals == case["rhs_evals"]
    assert rep.phi_iterations == case["phi_iterations"]
    assert rep.spectrum_rhs_evals == case["spectrum_rhs_evals"]
    assert [(s.dt, s.accepted, s.rhs_calls) for s in rep.steps] == \
        [(s["dt"], s["accepted"], s["rhs_calls"]) for s in case["steps"]]
    assert rep.checksum == case["checksum"]
    assert np.array_equal(rep.final, golden_io.arrays("run_cases")[f"{case['name']}__final"])
    assert rep.max_divb == case["max_divb"]


# ---- Krylov baseline (krylov.py) -------------------------------------------------

from oracle import krylov_np as kr  # noqa: E402


@pytest.mark.parametrize("case", golden_io.meta()["krylov"]["phi"], ids=lambda m: m["key"])
def test_oracle_krylov_phi(case):
    g = golden_io.arrays("krylov_cases")
    tag = case["case"]
    op, lin = _lin(g, case, tag)
    est = lj.power_alpha(lin, None, rng=np.random.default_rng(0))
    assert est.alpha == case["alpha"]
    calls = op.calls
    res = kr.phi_krylov(case["l"], lambda x: lj.fd_jvp(lin, x), g[f"{tag}__v"], case["dt"],
                        case["tol"], case["m_max"])
    assert (res.iterations, res.converged) == (case["iterations"], case["converged"])
    assert op.calls - calls == case["rhs_calls"]
    assert res.residual == case["residual"]
    assert np.array_equal(res.vector, g[case["key"]])


@pytest.mark.parametrize("case", golden_io.meta()["krylov"]["step"], ids=lambda m: m["name"])
def test_oracle_krylov_step(case):
    g = golden_io.arrays("krylov_cases")
    tag = case["name"]
    op, lin = _lin(g, case, tag)
    est = lj.power_alpha(lin, None, rng=np.random.default_rng(0))
    res = st.one_step(case["scheme"], op, lin.u, case["dt"], est, case["tol"], lin,
                      lj.CoeffCache(), method="krylov")
    assert res.converged == case["converged"]
    assert res.phi_iterations == case["phi_iterations"]
    assert res.error_estimate == case["error"]
    assert np.array_equal(res.new_state, g[f"{tag}__new"])


def test_oracle_krylov_errors():
    with pytest.raises(ValueError):
        kr.phi_krylov(1, lambda x: x, np.ones(4), 0.1, 0.0)
    with pytest.raises(ValueError):
        kr.phi_krylov(1, lambda x: x, np.ones(4), 0.1, 1e-8, m_max=201)
    with pytest.raises(ValueError):
        kr.phi_krylov(1, lambda x: x, np.zeros(4), 0.1, 1e-8)
    # J = -I: exact after one vector (happy breakdown), phi_1(-dt) v
    dt = 0.3
    res = kr.phi_krylov(1, lambda x: -x, np.arange(1.0, 5.0), dt, 1e-12)
    assert res.converged and res.iterations == 1 and res.residual == 0.0
    assert np.allclose(res.vector, np.arange(1.0, 5.0) * (1 - np.exp(-dt)) / dt, rtol=1e-13)


@pytest.mark.parametrize("case", golden_io.meta()["krylov"]["run"], ids=lambda m: m["name"])
def test_oracle_krylov_run(case):
    from paper_2108_13622_b200 import scenarios as sc
    setup = sc.kh_setup(case["nx"], t_final=case["t_final"])
    q = sc.initial_fields(setup)
    rep = st.run(q, setup.dx, setup.dy, setup.mu, setup.eta, setup.kappa,
                 case["scheme"], case["tol"], case["t_final"], cache=lj.CoeffCache(),
                 method="krylov")
    assert (rep.accepted, rep.rejected, rep.rhs_evals) == \
        (case["accepted"], case["rejected"], case["rhs_evals"])
    assert rep.checksum == case["checksum"]


# ---- walls, mu0 != 1, gamma != 5/3, Markstein spacings -----------------------------

@pytest.mark.parametrize("case", golden_io.meta()["leja_bc"], ids=lambda m: m["name"])
def test_oracle_leja_boundaries(case):
    g = golden_io.arrays("leja_bc_cases")
    tag = case["name"]
    q = g[f"{tag}__u"]

    def f(flat):
        return mhd_np.rhs(flat.reshape(q.shape), case["dx"], case["dy"], case["mu"],
                          case["eta"], case["kappa"], case["gamma"], case["mu0"],
                          case["periodic_x"], case["periodic_y"])

    op = lj.CountedRhs(f)
    lin = lj.Frozen(op, q.reshape(-1).copy())
    assert np.array_equal(lin.fu, g[f"{tag}__fu"])
    assert np.array_equal(lj.fd_jvp(lin, g[f"{tag}__w"]), g[f"{tag}__jw"])
    calls = op.calls
    est = lj.power_alpha(lin, None, rng=np.random.default_rng(0))
    assert (est.alpha, op.calls - calls) == (case["alpha"], case["power_calls"])
    for p in case["phi"]:
        res = lj.phi_leja(p["l"], lambda x: lj.fd_jvp(lin, x), g[f"{tag}__v"], p["dt"], p["q"],
                          p["theta"], p["tol"], lj.CoeffCache())
        assert (res.iterations, res.converged, res.residual) == \
            (p["iterations"], p["converged"], p["residual"])
        assert np.array_equal(res.vector, g[p["key"]])
