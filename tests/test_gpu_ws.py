"""The two-role register-split stencil kernel (stencil_ws_kernel, XMHD_WS=1)
against the one-role sliding-window kernel: F(u), J w and the first fused Leja term are
bitwise identical (same device functions, same operation order) on periodic
and reflecting grids, non-power-of-two spacings (Markstein divisions), mu0 != 1
(generic variant), the ideal (non-diffusive) operator and partial last column
strips.  XMHD_WS=0 at context creation selects the one-role kernel."""

import ctypes
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [
    # nx, ny, dx, dy, mu, eta, kappa, gamma, mu0, bcx, bcy
    (256, 64, 1 / 256, 2 / 64, 1e-3, 1e-3, 1e-3, 5 / 3, 1.0, 0, 0),
    (384, 50, 0.003125, 0.0051, 1e-3, 5e-3, 1e-3, 5 / 3, 1.0, 0, 0),
    (512, 40, 0.07, 0.11, 0.02, 0.01, 0.05, 1.4, 1.3, 1, 1),
    (300, 33, 0.05, 0.2, 0.0, 0.0, 0.0, 5 / 3, 1.0, 1, 0),
    (260, 29, 0.1, 0.15, 0.01, 0.02, 0.03, 5 / 3, 1.0, 0, 1),
]


def _state(rng, nx, ny):
    q = 0.1 * rng.standard_normal((8, ny, nx))
    q[0] = 1.0 + 0.1 * rng.standard_normal((ny, nx))
    q[7] = 6.0 + 0.1 * rng.standard_normal((ny, nx))
    return q


def _ctx(case, ws):
    from paper_2108_13622_b200 import _lib
    old = os.environ.get("XMHD_WS")
    os.environ["XMHD_WS"] = "1" if ws else "0"
    try:
        nx, ny, dx, dy, mu, eta, kappa, gamma, mu0, bcx, bcy = case
        return _lib.Context(nx, ny, dx, dy, mu, eta, kappa, gamma, mu0, bcx, bcy)
    finally:
        if old is None:
            os.environ.pop("XMHD_WS")
        else:
            os.environ["XMHD_WS"] = old


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}x{c[1]}_bc{c[9]}{c[10]}")
def test_ws_kernel_bitwise_vs_one_role(case):
    import torch
    from paper_2108_13622_b200 import _lib, leja
    lib = _lib.load()
    nx, ny = case[0], case[1]
    rng = np.random.default_rng(nx + ny)
    u = torch.from_numpy(_state(rng, nx, ny)).cuda().reshape(-1)
    w = torch.from_numpy(rng.standard_normal(8 * nx * ny)).cuda()
    ctx_ws, ctx_1 = _ctx(case, True), _ctx(case, False)
    out = {}
    for name, ctx in (("ws", ctx_ws), ("one", ctx_1)):
        h = ctx.bind_stream()
        f = torch.empty_like(u)
        assert lib.xmhd_rhs(h, _lib.ptr(u), _lib.ptr(f), None) == 0
        jw = torch.empty_like(u)
        called = ctypes.c_int()
        unorm = float(torch.linalg.norm(u))
        assert lib.xmhd_jvp(h, _lib.ptr(u), _lib.ptr(f), unorm, _lib.ptr(w), _lib.ptr(jw),
                            ctypes.byref(called), None, None) == 0
        # the first fused Leja term (its FD step comes from ||v||, not from a
        # stencil reduction, so y_1 and p_1 are comparable bit for bit)
        xi = np.ascontiguousarray(leja.leja_points(500))
        sh = leja.shift_and_scale(10.0)
        coeffs = np.ascontiguousarray(leja._compute_coeffs(1, sh.q, sh.theta, 64))
        dp = ctypes.POINTER(ctypes.c_double)
        assert lib.xmhd_leja_start_async(h, _lib.ptr(u), _lib.ptr(f), unorm, _lib.ptr(w),
                                         1e-3, sh.q, sh.theta, 1e-300, xi.ctypes.data_as(dp),
                                         coeffs.ctypes.data_as(dp), 64) == 0
        assert lib.xmhd_leja_launch(h, 1, 0) == 0
        st = _lib.LejaState()
        assert lib.xmhd_leja_sync(h, ctypes.byref(st)) == 0
        assert st.status == _lib.LEJA_RUNNING
        y1, p1 = torch.empty_like(u), torch.empty_like(u)
        assert lib.xmhd_leja_current_y(h, _lib.ptr(y1)) == 0
        assert lib.xmhd_leja_result(h, _lib.ptr(p1)) == 0
        torch.cuda.synchronize()
        out[name] = [t.cpu().numpy() for t in (f, jw, y1, p1)] + [st.ynorm]
    for k, what in enumerate(("F", "Jw", "y1", "p1")):
        assert np.array_equal(out["ws"][k], out["one"][k]), what
    # ||y_1||: two summation orders of the same values
    assert abs(out["ws"][4] - out["one"][4]) <= 1e-13 * out["one"][4]


def test_ws_plan_applies_to_the_bench_grid():
    from paper_2108_13622_b200 import _lib
    ctx = _ctx((2048, 2048, 1 / 2048, 2 / 2048, 1e-3, 1e-3, 1e-3, 5 / 3, 1.0, 0, 0), True)
    plan = ctx.plan()
    assert plan["grid"] <= 2 * 148 and plan["units"] >= plan["grid"]
