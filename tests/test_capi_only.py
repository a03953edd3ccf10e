"""The drop-in boundary exercised through ctypes ALONE, the way a non-Python
binder (or the reference's own ctypes stub in INTEGRATION.md) would use it:
the shared library is opened with ``ctypes.CDLL`` and typed here from the
header's declarations, with no helper from the package.  PyTorch only
allocates device memory.

* ``xmhd_newton_coeffs`` / ``xmhd_leja_schedule`` (host): bitwise the
  reference's ``_newton_coeffs`` chunks (leja.py:84-100, 119-130).
* ``xmhd_rhs`` / ``xmhd_jvp``: the ``bad_cells`` out-parameter carries the
  reference's ``RhsBlowupError`` payload (mhd.py:225-231).
* ``xmhd_leja``: one call = ``apply_phi_leja`` (leja.py:103-150) on golden
  cases of degree 11..170 (the 64 -> 128 -> 256 chunk growth included).
"""

import ctypes
import json
import os

import numpy as np
import pytest

import golden_io

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(REPO, "paper_2108_13622_b200", "_xmhd_b200.so")
FIELDS = ("rho", "mx", "my", "mz", "bx", "by", "bz", "en")
BAD_CELLS_LEN = 25

_P, _D, _I = ctypes.c_void_p, ctypes.c_double, ctypes.c_int
_PD, _PI = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)


@pytest.fixture(scope="module")
def so():
    from paper_2108_13622_b200 import build
    build.build_so()
    lib = ctypes.CDLL(SO)
    sigs = {
        "xmhd_create": [ctypes.POINTER(_P), _I, _I, _D, _D, _D, _D, _D, _D, _D, _I, _I, _P],
        "xmhd_destroy": [_P],
        "xmhd_rhs": [_P, _P, _P, _PI],
        "xmhd_jvp": [_P, _P, _P, _D, _P, _P, _PI, _PD, _PI],
        "xmhd_norm": [_P, _P, ctypes.c_longlong, _PD],
        "xmhd_leja": [_P, _I, _P, _P, _D, _P, _D, _D, _D, _D, _PD, _PD, _I, _P, _PI, _PI, _PD,
                      _PI, _PI],
        "xmhd_newton_coeffs": [_I, _D, _D, _PD, _I, _PD],
        "xmhd_leja_schedule": [_I, _D, _D, _PD, _PD],
    }
    _L = ctypes.c_longlong
    sigs.update({
        "xmhd_h2d_staged": [_P, _P, _L, _P],
        "xmhd_lincomb_diff": [_P, _P, _P, _L, ctypes.POINTER(_P), _PD, _I, _PD],
        "xmhd_lincomb_multi": [_P, ctypes.POINTER(_P), _I, _L, ctypes.POINTER(_P), _PD],
        "xmhd_stage_difference": [_P, _P, _P, _D, _P, _D, _P, _P, _PI, _PI],
        "xmhd_final_pair": [_P, _I, _P, _L, ctypes.POINTER(_P), _PD, _PD, _PI],
        "xmhd_diff_norms": [_P, _P, _P, _L, _PD],
        "xmhd_set_loop_kind": [_P, _I],
        "xmhd_leja_hint": [_P, _I],
        "xmhd_leja_start_inplace": [_P, _P, _P, _D, _P, _D, _D, _D, _D, _PD, _PD, _I],
        "xmhd_leja_set_pbuf": [_P, _P, _P],
        "xmhd_leja_set_dual_from": [_P, _I],
        "xmhd_leja_launch": [_P, _I, _I],
        "xmhd_leja_sync": [_P, _P],
        "xmhd_leja_result_inplace": [_P, _PI],
    })
    for name, args in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _I
    lib.xmhd_last_error.restype = ctypes.c_char_p
    lib.xmhd_last_error.argtypes = []
    return lib


def dptr(a):
    return a.ctypes.data_as(_PD)


def newton(so, l, q, theta, xi, count):
    out = np.empty(count)
    assert so.xmhd_newton_coeffs(l, q, theta, dptr(xi), count, dptr(out)) == 0
    return out


def test_newton_coeffs_and_schedule_bitwise(so):
    g = golden_io.arrays("coeff_cases")
    xi = np.ascontiguousarray(g["leja_points"])
    for m in golden_io.meta()["coeff"]:
        c = newton(so, m["l"], m["q"], m["theta"], xi, m["count"])
        assert np.array_equal(c, g[m["key"]]), m["key"]
    for l, adt in ((1, 10.0), (4, 100.0), (1, 300.0)):
        q, th = -0.5 * adt, 0.25 * adt
        table = np.empty(500)
        assert so.xmhd_leja_schedule(l, q, th, dptr(xi), dptr(table)) == 0
        lo = 0
        for size in (64, 128, 256, 500):
            assert np.array_equal(table[lo:size], newton(so, l, q, th, xi, size)[lo:size])
            lo = size
    bad = np.empty(4)
    assert so.xmhd_newton_coeffs(5, -1.0, 0.5, dptr(xi), 4, dptr(bad)) == 2
    assert so.xmhd_newton_coeffs(1, -1.0, 0.0, dptr(xi), 4, dptr(bad)) == 2


# ------------------------------------------------------------------ device

def _torch():
    import torch
    return torch


def dev(a):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def vp(t):
    return ctypes.c_void_p(t.data_ptr())


class Ctx:
    def __init__(self, so, nx, ny, dx, dy, mu, eta, kappa, gamma=5.0 / 3.0, mu0=1.0,
                 bcx=0, bcy=0):
        self.so = so
        self.h = _P()
        rc = so.xmhd_create(ctypes.byref(self.h), nx, ny, dx, dy, mu, eta, kappa, gamma, mu0,
                            bcx, bcy, None)
        assert rc == 0, so.xmhd_last_error()
        self.n = 8 * nx * ny

    def close(self):
        self.so.xmhd_destroy(self.h)


def cells_of(buf):
    out = []
    for k in range(8):
        f, i, j = buf[1 + 3 * k], buf[2 + 3 * k], buf[3 + 3 * k]
        if f < 0:
            break
        out.append((FIELDS[f], i, j))
    return buf[0], out


@pytest.mark.gpu
def test_rhs_bad_cells_are_the_reference_payload(so):
    torch = _torch()
    g = golden_io.arrays("rhs_cases")
    m = next(c for c in golden_io.meta()["rhs"] if c["name"] == "blowup")
    u = g["blowup__u"]
    ctx = Ctx(so, u.shape[2], u.shape[1], m["dx"], m["dy"], m["mu"], m["eta"], m["kappa"])
    try:
        ud = dev(u)
        f = torch.empty_like(ud)
        buf = (ctypes.c_int * BAD_CELLS_LEN)()
        assert so.xmhd_rhs(ctx.h, vp(ud), vp(f), buf) == 1
        count, cells = cells_of(buf)
        assert cells == [tuple(c) for c in m["cells"]]
        ref_count = int(m["message"].split(";")[1].split()[0])
        assert count == ref_count
        field, i, j = cells[0]
        assert m["message"] == (f"non-finite rhs in field {field} at cell (i={i}, j={j}); "
                                f"{count} cells affected")
        # NULL out-parameter: status only
        assert so.xmhd_rhs(ctx.h, vp(ud), vp(f), None) == 1
    finally:
        ctx.close()


@pytest.mark.gpu
def test_jvp_bad_cells_match_the_oracle(so):
    torch = _torch()
    from oracle import mhd_np
    g = golden_io.arrays("leja_cases")
    meta = next(c for c in golden_io.meta()["leja"] if c["name"] == "kh32")
    u = g["kh32__u"]
    ny, nx = u.shape[1:]
    w = np.array(g["kh32__w"]).reshape(u.shape)
    w[3, 5, 7] = np.inf          # ||w|| = inf -> eps = 0 -> u + 0*inf = nan (linearize.py:65-67)
    ctx = Ctx(so, nx, ny, meta["dx"], meta["dy"], meta["mu"], meta["eta"], meta["kappa"])
    try:
        ud, wd = dev(u), dev(w)
        fu = torch.empty_like(ud)
        assert so.xmhd_rhs(ctx.h, vp(ud), vp(fu), None) == 0
        out = torch.empty_like(ud)
        called = ctypes.c_int()
        buf = (ctypes.c_int * BAD_CELLS_LEN)()
        unorm = float(np.linalg.norm(u))
        rc = so.xmhd_jvp(ctx.h, vp(ud), vp(fu), unorm, vp(wd), vp(out), ctypes.byref(called),
                         None, buf)
        assert rc == 1 and called.value == 1
        x = u + 0.0 * w
        fx = mhd_np.rhs(x, meta["dx"], meta["dy"], meta["mu"], meta["eta"], meta["kappa"],
                        check=False)
        bad = np.argwhere(~np.isfinite(fx.reshape(u.shape)))
        count, cells = cells_of(buf)
        assert count == len(bad)
        assert cells == [(FIELDS[k], int(i), int(j)) for k, j, i in bad[:8]]
    finally:
        ctx.close()


def _leja_one_call(so, ctx, u, v, dt, q, theta, tol, xi, table):
    torch = _torch()
    ud, vd = dev(u), dev(v)
    fu = torch.empty_like(ud)
    assert so.xmhd_rhs(ctx.h, vp(ud), vp(fu), None) == 0
    un = ctypes.c_double()
    assert so.xmhd_norm(ctx.h, vp(ud), ud.numel(), ctypes.byref(un)) == 0
    p = torch.empty_like(ud)
    it, conv, calls = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    res = ctypes.c_double()
    buf = (ctypes.c_int * BAD_CELLS_LEN)()
    rc = so.xmhd_leja(ctx.h, 1, vp(ud), vp(fu), un.value, vp(vd), dt, q, theta, tol, dptr(xi),
                      dptr(table), table.size, vp(p), ctypes.byref(it), ctypes.byref(conv),
                      ctypes.byref(res), ctypes.byref(calls), buf)
    return rc, p.cpu().numpy(), it.value, bool(conv.value), res.value, calls.value


def _rel(a, b):
    a, b = np.ravel(a), np.ravel(b)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.gpu
def test_leja_one_call_matches_golden(so):
    xi = np.ascontiguousarray(golden_io.arrays("coeff_cases")["leja_points"])
    g = golden_io.arrays("leja_cases")
    for rec in golden_io.meta()["leja"]:
        name = rec["name"]
        u, v = g[f"{name}__u"], g[f"{name}__v"]
        ctx = Ctx(so, u.shape[2], u.shape[1], rec["dx"], rec["dy"], rec["mu"], rec["eta"],
                  rec["kappa"])
        try:
            for ph in rec["phi"]:
                if ph["l"] != 1:
                    continue
                table = np.empty(500)
                assert so.xmhd_leja_schedule(1, ph["q"], ph["theta"], dptr(xi),
                                             dptr(table)) == 0
                rc, p, it, conv, res, calls = _leja_one_call(
                    so, ctx, u, v, ph["dt"], ph["q"], ph["theta"], ph["tol"], xi, table)
                assert rc == 0, so.xmhd_last_error()
                assert (it, conv, calls) == (ph["iterations"], ph["converged"], ph["rhs_calls"])
                assert _rel(p, g[ph["key"]]) <= 1e-10, ph["key"]
        finally:
            ctx.close()


@pytest.mark.gpu
def test_leja_one_call_high_degree_and_short_table(so):
    """Degrees 84..170 cross the 64 and 128 chunk ends (leja.py:128-130) and a
    blow-up at the 256-chunk: same iteration counts and outcome as the
    reference, vectors within 10x the reference's own summation-order floor
    (tests/golden/large/degree.json)."""
    xi = np.ascontiguousarray(golden_io.arrays("coeff_cases")["leja_points"])
    meta = json.load(open(os.path.join(golden_io.GOLDEN, "large", "degree.json")))
    g = np.load(os.path.join(golden_io.GOLDEN, "large", "degree.npz"))
    for case in meta["cases"]:
        name = case["name"]
        u, v = g[f"{name}__u"], g[f"{name}__v"]
        ctx = Ctx(so, case["nx"], case["ny"], case["dx"], case["dy"], case["mu"], case["eta"],
                  case["kappa"])
        try:
            for ph in case["phi"]:
                if ph["l"] != 1:
                    continue
                table = np.empty(500)
                assert so.xmhd_leja_schedule(1, ph["q"], ph["theta"], dptr(xi),
                                             dptr(table)) == 0
                rc, p, it, conv, res, calls = _leja_one_call(
                    so, ctx, u, v, ph["dt"], ph["q"], ph["theta"], ph["tol"], xi, table)
                assert rc == 0, so.xmhd_last_error()
                assert (it, conv) == (ph["iterations"], ph["converged"]), ph["key"]
                assert calls == ph["rhs_calls"]
                if conv:
                    bound = max(1e-10, 10.0 * ph["floor_rel"])
                    assert _rel(p, g[ph["key"]]) <= bound, (ph["key"], _rel(p, g[ph["key"]]))
                else:
                    assert res == float("inf")
                # a table that ends before the degree reached is an error, never a truncation
                if ph["iterations"] > 70:
                    rc, *_ = _leja_one_call(so, ctx, u, v, ph["dt"], ph["q"], ph["theta"],
                                            ph["tol"], xi, np.ascontiguousarray(table[:64]))
                    assert rc == 2
                    assert b"coefficient table ended" in so.xmhd_last_error()
        finally:
            ctx.close()


class LejaState(ctypes.Structure):
    """xmhd_leja_state (include/xmhd_b200.h)."""
    _fields_ = [("status", _I), ("iterations", _I), ("rhs_calls", _I), ("m", _I),
                ("residual", _D), ("eps", _D), ("ynorm", _D)]


@pytest.mark.gpu
def test_stage_algebra_entry_points(so):
    """integrators.py:139-153 through the fewer-pass entry points, ctypes only:
    stage = u + c*p with d = stage - u and ||d|| from one call, then
    (F(stage) - F(u)) - jvp(d) from the JVP stencil's epilogue, against the same
    expression assembled from xmhd_rhs / xmhd_jvp outputs in NumPy (bit for
    bit), and the shared pass of the w_k combinations against NumPy."""
    torch = _torch()
    g = golden_io.arrays("leja_cases")
    meta = next(c for c in golden_io.meta()["leja"] if c["name"] == "kh32")
    u = np.array(g["kh32__u"])
    ny, nx = u.shape[1:]
    pvec = np.array(g["kh32__w"]).reshape(-1)
    ctx = Ctx(so, nx, ny, meta["dx"], meta["dy"], meta["mu"], meta["eta"], meta["kappa"])
    try:
        n = u.size
        # pageable upload through the staging pipeline
        ud = torch.empty(n, dtype=torch.float64, device="cuda")
        flat = np.ascontiguousarray(u.reshape(-1))
        assert so.xmhd_h2d_staged(vp(ud), flat.ctypes.data, flat.nbytes, None) == 0
        torch.cuda.synchronize()
        assert np.array_equal(ud.cpu().numpy(), flat)
        pd = dev(pvec)
        fu = torch.empty_like(ud)
        assert so.xmhd_rhs(ctx.h, vp(ud), vp(fu), None) == 0
        un = ctypes.c_double()
        assert so.xmhd_norm(ctx.h, vp(ud), n, ctypes.byref(un)) == 0
        # stage, d = stage - u, ||d||
        c = 0.37e-3
        stage, d = torch.empty_like(ud), torch.empty_like(ud)
        vecs = (_P * 4)(vp(ud), vp(pd), None, None)
        coef = (ctypes.c_double * 4)(1.0, c, 0.0, 0.0)
        dn = ctypes.c_double()
        assert so.xmhd_lincomb_diff(ctx.h, vp(stage), vp(d), n, vecs, coef, 2,
                                    ctypes.byref(dn)) == 0
        stage_ref = flat + c * pvec
        assert np.array_equal(stage.cpu().numpy(), stage_ref)
        assert np.array_equal(d.cpu().numpy(), stage_ref - flat)
        dn2 = ctypes.c_double()
        assert so.xmhd_norm(ctx.h, vp(d), n, ctypes.byref(dn2)) == 0
        assert dn.value == dn2.value
        # the stage difference: separate calls assembled on the host vs one fused tail
        fs, jd, out = torch.empty_like(ud), torch.empty_like(ud), torch.empty_like(ud)
        assert so.xmhd_rhs(ctx.h, vp(stage), vp(fs), None) == 0
        called = ctypes.c_int()
        assert so.xmhd_jvp(ctx.h, vp(ud), vp(fu), un.value, vp(d), vp(jd), ctypes.byref(called),
                           None, None) == 0
        assert called.value == 1
        ref = (fs.cpu().numpy() - fu.cpu().numpy()) - jd.cpu().numpy()
        assert so.xmhd_stage_difference(ctx.h, vp(ud), vp(fu), un.value, vp(d), dn.value, vp(fs),
                                        vp(out), ctypes.byref(called), None) == 0
        assert called.value == 1
        assert np.array_equal(out.cpu().numpy(), ref)
        # zero offset: jvp of zeros costs no RHS call (linearize.py:63-64)
        zero = torch.zeros_like(ud)
        assert so.xmhd_stage_difference(ctx.h, vp(ud), vp(fu), un.value, vp(zero), 0.0, vp(fs),
                                        vp(out), ctypes.byref(called), None) == 0
        assert called.value == 0
        assert np.array_equal(out.cpu().numpy(), fs.cpu().numpy() - fu.cpu().numpy())
        # w_k of EXPRB54s4 (integrators.py:186-189) in one pass
        a, b, cc = fs.cpu().numpy(), jd.cpu().numpy(), out.cpu().numpy()
        rows = ((64.0, -8.0, 0.0), (-60.0, -(285.0 / 8.0), 125.0 / 8.0),
                (0.0, 18.0, -(250.0 / 81.0)), (0.0, -60.0, 500.0 / 27.0))
        outs = [torch.empty_like(ud) for _ in rows]
        oarr = (_P * 4)(*[vp(o) for o in outs])
        varr = (_P * 3)(vp(fs), vp(jd), vp(out))
        flatc = (ctypes.c_double * 12)(*[x for r in rows for x in r])
        assert so.xmhd_lincomb_multi(ctx.h, oarr, 4, n, varr, flatc) == 0
        refs = (64.0 * a + -8.0 * b, (-60.0 * a + -(285.0 / 8.0) * b) + (125.0 / 8.0) * cc,
                18.0 * b + -(250.0 / 81.0) * cc, -60.0 * b + (500.0 / 27.0) * cc)
        for o, r in zip(outs, refs):
            assert np.array_equal(o.cpu().numpy(), r)
        assert so.xmhd_lincomb_multi(ctx.h, oarr, 5, n, varr, flatc) == 2   # XMHD_BADARG
        # the embedded pair of a step in one pass (integrators.py:168-171, 190-199):
        # the higher-order solution, ||lo - hi|| and ||hi|| as xmhd_diff_norms
        # reduces them on the materialised vectors
        dt = 0.0375
        h = [flat, a, b, cc, outs[0].cpu().numpy(), outs[1].cpu().numpy()]
        hv = [ud, fs, jd, out, outs[0], outs[1]]
        for scheme, nin in ((0, 4), (1, 6)):
            if scheme == 0:
                lo = (1.0 * h[0] + dt * h[1]) + dt * h[2]
                hi = 1.0 * lo + dt * h[3]
            else:
                lo = ((1.0 * h[0] + dt * h[1]) + dt * h[2]) + dt * h[3]
                hi = ((1.0 * h[0] + dt * h[1]) + dt * h[4]) + dt * h[5]
            varr6 = (_P * 6)(*[vp(x) for x in hv])
            c6 = (ctypes.c_double * 6)(1.0, dt, dt, dt, dt, dt)
            got = torch.empty_like(ud)
            err = (ctypes.c_double * 2)()
            bad = ctypes.c_int(-1)
            assert so.xmhd_final_pair(ctx.h, scheme, vp(got), n, varr6, c6, err,
                                      ctypes.byref(bad)) == 0
            assert np.array_equal(got.cpu().numpy(), hi) and bad.value == 0
            lo_d = torch.from_numpy(lo).cuda()
            two = (ctypes.c_double * 2)()
            assert so.xmhd_diff_norms(ctx.h, vp(lo_d), vp(got), n, two) == 0
            assert (err[0], err[1]) == (two[0], two[1])
            assert abs(err[0] - np.linalg.norm(lo - hi)) <= 1e-12 * err[0]
        hv[3] = torch.full_like(ud, float("inf"))
        varr6 = (_P * 6)(*[vp(x) for x in hv])
        assert so.xmhd_final_pair(ctx.h, 0, vp(got), n, varr6, c6, err, ctypes.byref(bad)) == 0
        assert bad.value == 1
        assert so.xmhd_final_pair(ctx.h, 7, vp(got), n, varr6, c6, err, ctypes.byref(bad)) == 2
    finally:
        ctx.close()


@pytest.mark.gpu
def test_leja_inplace_protocol_matches_the_one_call(so):
    """xmhd_leja_start_inplace + xmhd_leja_set_pbuf + xmhd_leja_launch (with the
    variant pairs of xmhd_leja_set_dual_from) + xmhd_leja_result_inplace on
    golden phi-calls: the reference's counters and vector, the caller's v left
    untouched, the result in one of the caller's two buffers, and the same bits
    with and without the variant pairs."""
    torch = _torch()
    xi = np.ascontiguousarray(golden_io.arrays("coeff_cases")["leja_points"])
    g = golden_io.arrays("leja_cases")
    rec = next(c for c in golden_io.meta()["leja"] if c["name"] == "kh32")
    u, v = g["kh32__u"], g["kh32__v"]
    ctx = Ctx(so, u.shape[2], u.shape[1], rec["dx"], rec["dy"], rec["mu"], rec["eta"],
              rec["kappa"])
    try:
        for ph in rec["phi"]:
            if ph["l"] != 1:
                continue
            table = np.empty(500)
            assert so.xmhd_leja_schedule(1, ph["q"], ph["theta"], dptr(xi), dptr(table)) == 0
            it, conv, calls = ph["iterations"], ph["converged"], ph["rhs_calls"]
            ud, vd = dev(u), dev(v)
            v_keep = vd.clone()
            fu = torch.empty_like(ud)
            assert so.xmhd_rhs(ctx.h, vp(ud), vp(fu), None) == 0
            un = ctypes.c_double()
            assert so.xmhd_norm(ctx.h, vp(ud), ud.numel(), ctypes.byref(un)) == 0
            pair = (torch.empty_like(ud), torch.empty_like(ud))
            first = None
            for dual_from in (0, 1, max(1, it - 3)):
                assert so.xmhd_leja_set_pbuf(ctx.h, vp(pair[0]), vp(pair[1])) == 0
                assert so.xmhd_leja_start_inplace(ctx.h, vp(ud), vp(fu), un.value, vp(vd),
                                                  ph["dt"], ph["q"], ph["theta"], ph["tol"],
                                                  dptr(xi), dptr(table), 500) == 0
                assert so.xmhd_leja_set_dual_from(ctx.h, dual_from) == 0
                st = LejaState()
                while True:
                    assert so.xmhd_leja_launch(ctx.h, 8, 0) == 0
                    assert so.xmhd_leja_sync(ctx.h, ctypes.byref(st)) == 0
                    if st.status != 0:
                        break
                which = ctypes.c_int(-1)
                assert so.xmhd_leja_result_inplace(ctx.h, ctypes.byref(which)) == 0
                torch.cuda.synchronize()
                assert which.value in (0, 1)
                assert (st.iterations, st.status == 1, st.rhs_calls) == (it, conv, calls)
                p = pair[which.value].cpu().numpy()
                assert _rel(p, g[ph["key"]]) <= 1e-10, ph["key"]
                if first is None:
                    first = (p.copy(), st.residual)
                else:   # the variant pairs change no bit
                    assert np.array_equal(p, first[0]) and st.residual == first[1]
                assert torch.equal(vd, v_keep)
                assert so.xmhd_leja_set_pbuf(ctx.h, None, None) == 0
    finally:
        ctx.close()


@pytest.mark.gpu
def test_leja_one_call_per_term_path_matches_golden(so):
    """xmhd_leja on the large-grid path (xmhd_set_loop_kind(ctx, 2): per-term
    launches with the in-place start and the variant pairs chosen from
    xmhd_leja_hint) on golden phi-calls of degree 11..170: the reference's
    counters and vectors whatever the hint, and the same bits for every hint."""
    xi = np.ascontiguousarray(golden_io.arrays("coeff_cases")["leja_points"])
    meta = json.load(open(os.path.join(golden_io.GOLDEN, "large", "degree.json")))
    g = np.load(os.path.join(golden_io.GOLDEN, "large", "degree.npz"))
    seen = 0
    for case in meta["cases"]:
        name = case["name"]
        u, v = g[f"{name}__u"], g[f"{name}__v"]
        ctx = Ctx(so, case["nx"], case["ny"], case["dx"], case["dy"], case["mu"], case["eta"],
                  case["kappa"])
        try:
            assert so.xmhd_set_loop_kind(ctx.h, 2) == 0
            for ph in case["phi"]:
                if ph["l"] != 1:
                    continue
                table = np.empty(500)
                assert so.xmhd_leja_schedule(1, ph["q"], ph["theta"], dptr(xi),
                                             dptr(table)) == 0
                first = None
                for hint in (2, ph["iterations"] + 1, 400):
                    assert so.xmhd_leja_hint(ctx.h, hint) == 0
                    rc, p, it, conv, res, calls = _leja_one_call(
                        so, ctx, u, v, ph["dt"], ph["q"], ph["theta"], ph["tol"], xi, table)
                    assert rc == 0, so.xmhd_last_error()
                    assert (it, conv, calls) == (ph["iterations"], ph["converged"],
                                                 ph["rhs_calls"]), (ph["key"], hint)
                    if conv:
                        bound = max(1e-10, 10.0 * ph["floor_rel"])
                        assert _rel(p, g[ph["key"]]) <= bound, ph["key"]
                    if first is None:
                        first = (p.copy(), res)
                    else:
                        assert np.array_equal(p, first[0]) and res == first[1], (ph["key"], hint)
                    seen += 1
        finally:
            ctx.close()
    assert seen >= 6
