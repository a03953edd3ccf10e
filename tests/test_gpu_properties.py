"""Size-independent properties of the hot path at the BENCHMARKED sizes, where
no CPU oracle finishes: exact symmetries of the discrete
operators that hold bit for bit in IEEE arithmetic.

* Translation equivariance of mhd_rhs on a periodic grid (the reference's own
  tests/test_mhd.py:63-70 checks it on small grids): F(roll(u)) == roll(F(u))
  for shifts that cross the kernel's column strips and row segments.
* Positive power-of-two homogeneity of the FD-JVP (linearize.py:62-67): for
  w' = 2^k w the FD step is eps' = eps / 2^k, so u + eps'*w' is the same state
  bit for bit and (F - F(u)) / eps' = 2^k (F - F(u)) / eps exactly.
* The same homogeneity through a whole Leja phi-action (leja.py:116-148)
  while every interpolant has norm >= 1: every Newton basis vector, the
  interpolant and the norms scale by 2^k and the residuals
  |c_m| ||y_m|| / max(1, ||p_m||) do not, so the call takes the same
  iterations and returns 2^k p.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


_CACHE = {}


def _setup(n, kind):
    """(module, setup, device state, MhdRhs), built once per grid for the file."""
    key = (n, kind)
    if key not in _CACHE:
        _CACHE.clear()   # one large state at a time
        _CACHE[key] = _build(n, kind)
    return _CACHE[key]


def _build(n, kind):
    import paper_2108_13622_b200 as xb
    from paper_2108_13622_b200 import scenarios as sc
    s = sc.CONFIGS[1]() if kind == "kh" else sc.CONFIGS[4]()
    s.nx = s.ny = n
    q = sc.initial_fields(s)
    u = torch.from_numpy(q).cuda()
    st = xb.StateGrid(n, n, s.dx, s.dy, u)
    mhd = xb.MhdRhs(st, xb.MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa))
    return xb, s, u, mhd


@pytest.mark.parametrize("n,kind", [(2048, "kh"), (8192, "harris")])
def test_rhs_translation_equivariance_full_size(n, kind):
    xb, s, u, mhd = _setup(n, kind)
    f = mhd(u.reshape(-1)).reshape(u.shape)
    for dy, dx in ((0, 1), (1, 0), (61, 125), (n // 2 + 3, 977)):
        ur = torch.roll(u, shifts=(dy, dx), dims=(1, 2)).contiguous()
        fr = mhd(ur.reshape(-1)).reshape(u.shape)
        assert torch.equal(fr, torch.roll(f, shifts=(dy, dx), dims=(1, 2))), (dy, dx)


@pytest.mark.parametrize("n,kind", [(8192, "harris"), (2048, "kh")])
def test_jvp_power_of_two_homogeneity_full_size(n, kind):
    xb, s, u, mhd = _setup(n, kind)
    lin = xb.FrozenLinearization(xb.RhsOperator(mhd), u.reshape(-1))
    w = torch.from_numpy(sc_unit(u.numel(), 5)).cuda()
    jw = xb.jvp(lin, w)
    for k in (1, 3, -2):
        jk = xb.jvp(lin, w * 2.0 ** k)
        assert torch.equal(jk, jw * 2.0 ** k), k


def sc_unit(n, seed):
    from paper_2108_13622_b200 import scenarios as sc
    return sc.unit_gaussian(n, seed)


def test_leja_power_of_two_homogeneity_bench_size():
    """The bench workload (2048^2, alpha*dt = 10 and 100) with v scaled to
    ||v|| = 64 and 256 (so max(1, ||p_m||) = ||p_m|| throughout):
    phi_1(dt J)(256 v) == 4 phi_1(dt J)(64 v) bit for bit, same iterations
    and residuals."""
    from paper_2108_13622_b200 import leja
    xb, s, u, mhd = _setup(2048, "kh")
    lin = xb.FrozenLinearization(xb.RhsOperator(mhd), u.reshape(-1))
    alpha = 5875.808769779558
    v = torch.from_numpy(sc_unit(u.numel(), 2)).cuda()
    for adt in (10.0, 100.0):
        dt = adt / alpha
        sh = xb.shift_and_scale(alpha * dt)
        leja._coeff_cache.clear()
        r1 = xb.apply_phi_leja(1, xb.JacobianAction(lin), v * 64.0, dt, sh, 1e-10)
        leja._coeff_cache.clear()
        r2 = xb.apply_phi_leja(1, xb.JacobianAction(lin), v * 256.0, dt, sh, 1e-10)
        assert (r1.iterations, r1.converged) == (r2.iterations, r2.converged)
        assert r1.residual == r2.residual
        assert torch.equal(r2.vector, r1.vector * 4.0), adt


def test_driver_variants_agree_at_the_bench_size():
    """The bench workload (2048^2, alpha*dt = 10 and 100, tol 1e-10) through
    every host-paced driver variant -- copying start / copy-out vs in-place
    start / result hand-off, plain odd/even schedule vs variant pairs near the
    expected end -- gives the same vector bit for bit, the same degree,
    residual and coefficient cache."""
    from paper_2108_13622_b200 import leja
    xb, s, u, mhd = _setup(2048, "kh")
    lin = xb.FrozenLinearization(xb.RhsOperator(mhd), u.reshape(-1))
    alpha = 5875.808769779558
    v = torch.from_numpy(sc_unit(u.numel(), 2)).cuda()
    old = (leja.ZERO_COPY, leja.ADAPTIVE)
    try:
        for adt in (10.0, 100.0):
            dt = adt / alpha
            sh = xb.shift_and_scale(alpha * dt)
            ref = None
            for zc, ad in ((False, False), (True, False), (True, True), (False, True)):
                leja.ZERO_COPY, leja.ADAPTIVE = zc, ad
                leja._coeff_cache.clear()
                r = xb.apply_phi_leja(1, xb.JacobianAction(lin), v, dt, sh, 1e-10)
                keys = [(k, c.size) for k, c in leja._coeff_cache.items()]
                if ref is None:
                    ref = (r, keys)
                    assert r.converged
                    continue
                assert (r.iterations, r.converged, r.residual) == \
                    (ref[0].iterations, ref[0].converged, ref[0].residual), (adt, zc, ad)
                assert keys == ref[1]
                assert torch.equal(r.vector, ref[0].vector), (adt, zc, ad)
    finally:
        leja.ZERO_COPY, leja.ADAPTIVE = old


@pytest.mark.parametrize("n", [4096])
def test_fused_stage_algebra_at_config3_size(n):
    """One EXPRB43 step of config 3's state (KH 4096^2): the fused stage
    algebra (stage + offset + norm in one kernel, the JVP epilogue's stage
    difference, the shared w_k pass) against one kernel per reference
    expression -- same new state bit for bit, same error estimate and counters."""
    from paper_2108_13622_b200 import integrators, leja
    xb, s, u, mhd = _setup(n, "kh")
    op = xb.RhsOperator(mhd)
    uf = u.reshape(-1)
    alpha = 5875.808769779558 * (n / 2048.0) ** 2
    dt = 4.0 / alpha
    old = integrators.FUSE_STAGES
    res = []
    try:
        for fuse in (False, True):
            integrators.FUSE_STAGES = fuse
            leja._coeff_cache.clear()
            lin = xb.FrozenLinearization(op, uf)
            c0 = op.calls
            r = xb.step(xb.Scheme.EXPRB43, op, uf, dt, alpha=alpha, tol=1e-6, lin=lin)
            res.append((r, op.calls - c0))
    finally:
        integrators.FUSE_STAGES = old
    (a, ca), (b, cb) = res
    assert a.converged and (a.rhs_calls, a.phi_iterations, a.phi_applications, ca) == \
        (b.rhs_calls, b.phi_iterations, b.phi_applications, cb)
    assert a.error_estimate == b.error_estimate
    assert torch.equal(a.new_state, b.new_state)


def test_stream_kernels_at_full_size():
    """The stage-algebra stream kernels on 8192^2-sized vectors (4.3 GB each):
    exact power-of-two homogeneity (2^k scales every rounding exactly), the
    flagged combination's norm equal to the norm kernel's, and a strided sample
    of every output against the same NumPy expression, bit for bit."""
    from paper_2108_13622_b200 import _ops
    _CACHE.clear()
    torch.cuda.empty_cache()
    n = 8 * 8192 * 8192
    g = torch.Generator(device="cuda").manual_seed(7)
    vs = [torch.randn(n, dtype=torch.float64, device="cuda", generator=g) for _ in range(3)]
    idx = torch.arange(0, n, 99991, device="cuda")
    host = [v[idx].cpu().numpy() for v in vs]
    cs = (1.0, 0.37, -2.5)
    out, nrm, bad = _ops.lincomb(cs, vs, want_norm=True)
    assert not bad and nrm == _ops.norm(out)
    assert np.array_equal(out[idx].cpu().numpy(), (cs[0] * host[0] + cs[1] * host[1]) + cs[2] * host[2])
    out4 = _ops.lincomb(tuple(4.0 * c for c in cs), vs)
    out.mul_(4.0)
    assert torch.equal(out4, out)
    del out4, out
    st, d, dn = _ops.lincomb_diff(cs, vs)
    ref = (host[0] + cs[1] * host[1]) + cs[2] * host[2]
    assert np.array_equal(st[idx].cpu().numpy(), ref)
    assert np.array_equal(d[idx].cpu().numpy(), ref - host[0])
    assert dn == _ops.norm(d)
    del st, d
    rows = ((64.0, -8.0, 0.0), (0.0, 18.0, -(250.0 / 81.0)))
    w = _ops.lincomb_multi(rows, vs)
    assert np.array_equal(w[0][idx].cpu().numpy(), 64.0 * host[0] + -8.0 * host[1])
    assert np.array_equal(w[1][idx].cpu().numpy(), 18.0 * host[1] + -(250.0 / 81.0) * host[2])
    assert _ops.norm(vs[0] * 8.0) == 8.0 * _ops.norm(vs[0])
