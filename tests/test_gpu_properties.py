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
