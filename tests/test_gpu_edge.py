"""GPU edge cases of the hot path against the CPU oracle / dense references.

Mirrors the reference's own test strategy (pkg/tests/test_mhd.py,
test_leja.py, test_linearize.py, test_integrators.py): zero vectors, non-finite
states, underestimated spectra, reflecting walls, mu0 != 1, dense-matrix
oracles for the generic matvec path, invariants of the RHS.
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = a.cpu().numpy() if torch.is_tensor(a) else np.asarray(a)
    b = b.cpu().numpy() if torch.is_tensor(b) else np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _mhd(nx=24, ny=20, refl=False, mu0=1.0, seed=3):
    import paper_2108_13622_b200 as xb
    from oracle import leja_np as olj, mhd_np
    rng = np.random.default_rng(seed)
    q = 0.1 * rng.standard_normal((8, ny, nx))
    q[0] = 1.0 + 0.1 * rng.standard_normal((ny, nx))
    q[7] = 6.0 + 0.1 * rng.standard_normal((ny, nx))
    dx, dy = 0.08, 0.11
    prm = dict(mu=0.02, eta=0.03, kappa=0.05)
    bcy = xb.Boundary.REFLECTING if refl else xb.Boundary.PERIODIC
    params = xb.MHDParams(mu0=mu0, bc_y=bcy, **prm)
    st = xb.StateGrid(nx, ny, dx, dy, torch.from_numpy(q).cuda())
    op = xb.RhsOperator(xb.MhdRhs(st, params))
    lin = xb.FrozenLinearization(op, st.flat())

    def f(flat):
        return mhd_np.rhs(flat.reshape(q.shape), dx, dy, mu0=mu0, periodic_y=not refl, **prm)
    oop = olj.CountedRhs(f)
    olin = olj.Frozen(oop, q.reshape(-1))
    return xb, q, op, lin, oop, olin


def test_zero_vector_phi_fused():
    from oracle import leja_np as olj
    xb, q, op, lin, oop, olin = _mhd()
    sh = xb.shift_and_scale(5.0)
    calls = op.calls
    res = xb.apply_phi_leja(1, xb.JacobianAction(lin), torch.zeros(q.size, dtype=torch.float64,
                                                                    device="cuda"), 0.1, sh, 1e-10)
    ref = olj.phi_leja(1, lambda x: olj.fd_jvp(olin, x), np.zeros(q.size), 0.1, sh.q, sh.theta,
                       1e-10, olj.CoeffCache())
    assert res.converged and res.iterations == ref.iterations == 2
    assert op.calls == calls    # zero directions cost no RHS evaluation
    assert torch.count_nonzero(res.vector) == 0


def test_nonfinite_direction_raises_like_reference():
    from oracle import leja_np as olj, mhd_np
    xb, q, op, lin, oop, olin = _mhd()
    v = np.ones(q.size)
    v[17] = np.nan
    sh = xb.shift_and_scale(5.0)
    with pytest.raises(mhd_np.NonFiniteRhs) as ref_err:
        olj.phi_leja(1, lambda x: olj.fd_jvp(olin, x), v, 0.1, sh.q, sh.theta, 1e-10,
                     olj.CoeffCache())
    calls = op.calls
    with pytest.raises(xb.RhsBlowupError) as err:
        xb.apply_phi_leja(1, xb.JacobianAction(lin), torch.from_numpy(v).cuda(), 0.1, sh, 1e-10)
    assert str(err.value) == str(ref_err.value)
    assert err.value.cells == ref_err.value.cells
    assert op.calls == calls + 1


def test_underestimated_spectrum_reports_nonconvergence():
    from oracle import leja_np as olj
    xb, q, op, lin, oop, olin = _mhd()
    alpha = olj.power_alpha(olin, None, rng=np.random.default_rng(0)).alpha
    v = np.random.default_rng(1).standard_normal(q.size)
    dt = 50.0 / alpha
    sh = xb.shift_and_scale(1e-3 * alpha * dt)      # interval far too small
    res = xb.apply_phi_leja(1, xb.JacobianAction(lin), torch.from_numpy(v).cuda(), dt, sh, 1e-10)
    ref = olj.phi_leja(1, lambda x: olj.fd_jvp(olin, x), v, dt, sh.q, sh.theta, 1e-10,
                       olj.CoeffCache())
    assert not res.converged and not ref.converged
    assert res.iterations == ref.iterations
    assert res.residual == ref.residual == math.inf


@pytest.mark.parametrize("refl,mu0", [(True, 1.0), (False, 1.3), (True, 0.7)])
def test_phi_and_step_reflecting_and_mu0(refl, mu0):
    from oracle import leja_np as olj, steppers_np as ost
    from paper_2108_13622_b200 import leja
    xb, q, op, lin, oop, olin = _mhd(refl=refl, mu0=mu0)
    assert np.array_equal(lin.base_rhs.cpu().numpy(), olin.fu)
    est = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0))
    oest = olj.power_alpha(olin, None, rng=np.random.default_rng(0))
    assert abs(est.alpha - oest.alpha) <= 1e-10 * oest.alpha
    v = np.random.default_rng(2).standard_normal(q.size)
    for l, adt in ((1, 1.0), (3, 8.0)):
        dt = adt / oest.alpha
        sh = xb.shift_and_scale(oest.alpha * dt)
        leja._coeff_cache.clear()
        res = xb.apply_phi_leja(l, xb.JacobianAction(lin), torch.from_numpy(v).cuda(), dt, sh,
                                1e-10)
        ref = olj.phi_leja(l, lambda x: olj.fd_jvp(olin, x), v, dt, sh.q, sh.theta, 1e-10,
                           olj.CoeffCache())
        assert res.iterations == ref.iterations and res.converged == ref.converged
        assert rel(res.vector, ref.vector) <= 1e-10
    leja._coeff_cache.clear()
    dt = 0.2 / oest.alpha
    res = xb.step(xb.Scheme.EXPRB43, op, lin.base_state, dt, alpha=oest.alpha, tol=1e-6, lin=lin)
    ref = ost.one_step("exprb43", oop, olin.u, dt, oest.alpha, 1e-6, olin, olj.CoeffCache())
    assert res.rhs_calls == ref.rhs_calls and res.phi_iterations == ref.phi_iterations
    assert rel(res.new_state, ref.new_state) <= 1e-10


def _phi_dense(l, a):
    from scipy.linalg import expm
    n = a.shape[0]
    if l == 0:
        return expm(a)
    m = np.zeros((n * (l + 1), n * (l + 1)))
    m[:n, :n] = a
    for k in range(l):
        m[k * n:(k + 1) * n, (k + 1) * n:(k + 2) * n] = np.eye(n)
    return expm(m)[:n, l * n:]


def _neg_spectrum(rng, n, lo=-20.0):
    eig = rng.uniform(lo, 0.0, n)
    qm, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return qm @ np.diag(eig) @ qm.T


@pytest.mark.parametrize("l", [0, 1, 3, 4])
def test_generic_matvec_dense_oracle(l):
    import paper_2108_13622_b200 as xb
    rng = np.random.default_rng(100 + l)
    for _ in range(3):
        a = _neg_spectrum(rng, 32)
        v = rng.standard_normal(32)
        exact = _phi_dense(l, a) @ v
        res = xb.apply_phi_leja(l, lambda w: a @ w, v, 1.0, xb.shift_and_scale(25.0), 1e-10)
        assert res.converged
        assert rel(res.vector, exact) <= 1e-8


def test_generic_matvec_linearity_and_cost():
    import paper_2108_13622_b200 as xb
    rng = np.random.default_rng(5)
    a = _neg_spectrum(rng, 24)
    v, w = rng.standard_normal(24), rng.standard_normal(24)
    sh = xb.shift_and_scale(25.0)
    calls = [0]

    def mv(x):
        calls[0] += 1
        return a @ x
    rv = xb.apply_phi_leja(1, mv, v, 1.0, sh, 1e-11)
    assert calls[0] == rv.iterations
    rw = xb.apply_phi_leja(1, lambda x: a @ x, w, 1.0, sh, 1e-11)
    rc = xb.apply_phi_leja(1, lambda x: a @ x, 2.0 * v - 3.0 * w, 1.0, sh, 1e-11)
    combo = 2.0 * rv.vector - 3.0 * rw.vector
    assert np.linalg.norm(rc.vector - combo) <= 100 * 1e-11 * max(1.0, np.linalg.norm(rc.vector))
    loose = xb.apply_phi_leja(1, lambda x: a @ x, v, 1.0, sh, 1e-6)
    assert loose.residual >= rv.residual


def test_exprb43_linear_exactness_generic():
    import paper_2108_13622_b200 as xb
    from scipy.linalg import expm
    rng = np.random.default_rng(30)
    a = _neg_spectrum(rng, 40, lo=-8.0)
    op = xb.RhsOperator(lambda u: a @ u, host=True)
    u = rng.standard_normal(40)
    res = xb.step(xb.Scheme.EXPRB43, op, u, 0.4, alpha=10.0, tol=1e-11)
    assert res.converged and res.phi_applications == 5
    assert res.rhs_calls == 5 + res.phi_iterations
    assert xb.error_norm(res.new_state, expm(0.4 * a) @ u) <= 1e-6


def test_step_nonconvergence_propagates():
    import paper_2108_13622_b200 as xb
    a = np.diag([-5000.0, -1.0])
    op = xb.RhsOperator(lambda u: a @ u, host=True)
    res = xb.step(xb.Scheme.EXPRB43, op, np.array([1.0, 1.0]), 1.0, alpha=1.0, tol=1e-10)
    assert not res.converged


def test_rhs_invariants():
    """Reference invariants: uniform state -> 0, translation equivariance (bitwise),
    discrete div B of the induction rate vanishes (test_mhd.py:28-31, 63-70, 108-119)."""
    import paper_2108_13622_b200 as xb
    g = xb.StateGrid.zeros(16, 12, 0.1, 0.15)
    g.data[0], g.data[1], g.data[2], g.data[3] = 1.3, 0.4, -0.2, 0.7
    g.data[4], g.data[5], g.data[6], g.data[7] = 0.5, -0.3, 2.0, 5.0
    assert np.abs(xb.mhd_rhs(g, xb.MHDParams(0.1, 0.05, 0.2))).max() <= 1e-13
    rng = np.random.default_rng(3)
    q = 0.1 * rng.standard_normal((8, 16, 16))
    q[0] += 1.0
    q[7] += 6.0
    params = xb.MHDParams(mu=0.03, eta=0.02, kappa=0.1)
    base = xb.mhd_rhs(xb.StateGrid(16, 16, 0.1, 0.1, q), params).reshape(8, 16, 16)
    rolled = xb.mhd_rhs(xb.StateGrid(16, 16, 0.1, 0.1, np.roll(q, 1, axis=2)), params)
    assert np.array_equal(np.roll(base, 1, axis=2), rolled.reshape(8, 16, 16))
    gdot = np.zeros((8, 16, 16))
    gdot[4], gdot[5] = base[4], base[5]
    div = xb.discrete_div_b(xb.StateGrid(16, 16, 0.1, 0.1, gdot), params)
    scale = max(np.abs(base[4]).max(), np.abs(base[5]).max()) / 0.1
    assert np.abs(div).max() <= 1e-12 * max(1.0, scale)


def test_checkpoint_roundtrip(tmp_path):
    import paper_2108_13622_b200 as xb
    from oracle import mhd_np
    rng = np.random.default_rng(37)
    q = rng.standard_normal((8, 7, 12))
    st = xb.StateGrid(12, 7, 0.05, 0.08, torch.from_numpy(q).cuda())
    path = tmp_path / "state.chk"
    xb.write_checkpoint(path, st, 1.25)
    assert path.read_bytes() == mhd_np.checkpoint_bytes(q, 0.05, 0.08, 1.25)
    loaded, t = xb.read_checkpoint(path)
    assert t == 1.25 and np.array_equal(loaded.data, q)


def _host_power(xb, lin, w0, prev=None):
    from paper_2108_13622_b200 import linearize
    old = linearize._HOST_POWER
    linearize._HOST_POWER = True
    try:
        if prev is not None:
            return xb.estimate_alpha(lin, prev)
        return xb.estimate_alpha(lin, None, rng=np.random.default_rng(w0))
    finally:
        linearize._HOST_POWER = old


@pytest.mark.parametrize("refl,mu0", [(False, 1.0), (True, 0.7)])
def test_device_power_iteration_matches_host_loop_and_oracle(refl, mu0):
    """xmhd_power (one device-resident loop) against the host loop over the
    fused JVP and the NumPy oracle (linearize.py:113-135): same iteration
    count and RHS calls, alpha and the warm-start vector within rounding of
    the norm summation order; then a warm-started refresh."""
    from oracle import leja_np as olj
    xb, q, op, lin, oop, olin = _mhd(refl=refl, mu0=mu0)
    c0 = op.calls
    dev = xb.estimate_alpha(lin, None, rng=np.random.default_rng(5))
    c1 = op.calls
    host = _host_power(xb, lin, 5)
    c2 = op.calls
    ocalls = oop.calls
    ref = olj.power_alpha(olin, None, rng=np.random.default_rng(5))
    assert c1 - c0 == c2 - c1 == oop.calls - ocalls == len(ref.mags)
    assert len(dev.mags) == len(host.mags) == len(ref.mags)
    assert abs(dev.alpha - ref.alpha) <= 1e-12 * ref.alpha
    assert abs(dev.alpha - host.alpha) <= 1e-13 * host.alpha
    assert rel(dev.vector, ref.vector) <= 1e-10
    # warm start from the previous vector once the cache expires (linearize.py:108-109)
    stale = xb.SpectralEstimate(alpha=dev.alpha, age_steps=dev.interval - 1, vector=dev.vector)
    ostale = olj.Spectrum(ref.alpha, ref.interval - 1, ref.interval, ref.safety, ref.vector,
                          ref.mags)
    dev2 = xb.estimate_alpha(lin, stale)
    ref2 = olj.power_alpha(olin, ostale)
    assert len(dev2.mags) == len(ref2.mags)
    assert abs(dev2.alpha - ref2.alpha) <= 1e-12 * ref2.alpha
    assert torch.equal(stale.vector, dev.vector)    # the start vector is not mutated


def test_device_power_zero_start_and_zero_operator():
    """A zero start vector restarts from ones (linearize.py:115-116); a zero
    Jacobian (uniform state, F = 0 and J w = 0) gives alpha 0 and no vector."""
    from oracle import leja_np as olj
    xb, q, op, lin, oop, olin = _mhd()
    zero = xb.SpectralEstimate(alpha=1.0, age_steps=49,
                               vector=torch.zeros(q.size, dtype=torch.float64, device="cuda"))
    dev = xb.estimate_alpha(lin, zero)
    ref = olj.power_alpha(olin, olj.Spectrum(1.0, 49, 50, 1.25, np.zeros(q.size), []))
    assert len(dev.mags) == len(ref.mags)
    assert abs(dev.alpha - ref.alpha) <= 1e-12 * ref.alpha
    # uniform state, uniform direction: u + eps*w is uniform, so F(u + eps*w) = F(u) = 0
    # exactly, J w = 0, magnitude 0 -> alpha 0 and no vector after one RHS call
    u = np.zeros((8, 12, 16))
    u[0] = 1.0
    u[7] = 2.0
    st = xb.StateGrid(16, 12, 0.1, 0.1, torch.from_numpy(u).cuda())
    op2 = xb.RhsOperator(xb.MhdRhs(st, xb.MHDParams(mu=0.01, eta=0.01, kappa=0.01)))
    lin2 = xb.FrozenLinearization(op2, st.flat())
    c = op2.calls
    ones = xb.SpectralEstimate(alpha=1.0, age_steps=49,
                               vector=torch.ones(u.size, dtype=torch.float64, device="cuda"))
    est = xb.estimate_alpha(lin2, ones)
    assert est.alpha == 0.0 and est.vector is None and op2.calls == c + 1


def test_device_power_nonfinite_rhs_raises_like_reference():
    """A NaN in the start vector makes u + eps*w non-finite: the power iteration raises
    RhsBlowupError with the reference's message and cells (mhd.py:225-231)."""
    from oracle import leja_np as olj, mhd_np
    xb, q, op, lin, oop, olin = _mhd()
    w = np.ones(q.size)
    w[33] = np.nan      # ||w|| = nan: every iterate and eps are nan, F(u + eps*w) is not finite
    prev_ref = olj.Spectrum(1.0, 49, 50, 1.25, w, [])
    with pytest.raises(mhd_np.NonFiniteRhs) as ref_err:
        olj.power_alpha(olin, prev_ref)
    calls = op.calls
    prev = xb.SpectralEstimate(alpha=1.0, age_steps=49, vector=torch.from_numpy(w).cuda())
    with pytest.raises(xb.RhsBlowupError) as err:
        xb.estimate_alpha(lin, prev)
    assert str(err.value) == str(ref_err.value)
    assert err.value.cells == ref_err.value.cells
    assert op.calls == calls + 1


def test_prefetched_start_vector_uploaded_and_identical():
    """On a GPU the prefetched start vector is drawn in chunks and uploaded as
    it goes (device-resident when the first estimate needs it); values and the
    continuation of the run RNG's stream are still exactly the reference's."""
    from paper_2108_13622_b200 import harness
    for n in (1_000_003, 2 * harness._PrefetchedNormals._CHUNK + 5, 9_000_011):
        pre = harness._PrefetchedNormals(5, n)
        ref = np.random.default_rng(5)
        w = pre.standard_normal(n)
        assert torch.is_tensor(w) and w.is_cuda and w.numel() == n
        assert np.array_equal(w.cpu().numpy(), ref.standard_normal(n))
        assert np.array_equal(pre.standard_normal(9), ref.standard_normal(9))


def test_staged_pageable_h2d_is_exact():
    """Large pageable NumPy inputs go through the page-locked staging pipeline
    (_ops._Staging, several 32 MB chunks, a partial last chunk): bitwise the
    plain copy, for NumPy arrays and pageable CPU tensors, repeated calls."""
    import numpy as np
    import torch
    from paper_2108_13622_b200 import _ops
    rng = np.random.default_rng(3)
    for n in (2 * (1 << 20) + 5, 9 * (1 << 20) + 123):
        a = rng.standard_normal(n)
        for _ in range(2):
            d = _ops.as_device(a)
            assert d.is_cuda and d.shape == a.shape
            assert torch.equal(d.cpu(), torch.from_numpy(a))
        t = torch.from_numpy(a[: (n // 5) * 5].reshape(-1, 5))
        d2 = _ops.as_device(t)
        assert d2.shape == t.shape and torch.equal(d2.cpu(), t)
