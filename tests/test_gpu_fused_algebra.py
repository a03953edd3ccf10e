"""The passes saved around the fused stencil: vectorised stream kernels, the
fused stage algebra of the exponential Rosenbrock steps, and the zero-copy
start / result of a host-paced Leja call.  All of them must be invisible:
the same operations in the same order as the reference's expressions
(integrators.py:139-199, leja.py:121-148), so every comparison here is
bit for bit against NumPy or against the one-kernel-per-expression path.
"""

import contextlib
import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _views(n, k, seed, misalign):
    """k device vectors of n doubles; with `misalign` they start 8 bytes off a
    16-byte boundary (the kernels then take their 64-bit path)."""
    rng = np.random.default_rng(seed)
    host = [rng.standard_normal(n) for _ in range(k)]
    dev = []
    for h in host:
        buf = torch.empty(n + 2, dtype=torch.float64, device="cuda")
        off = 1 if misalign else 0
        v = buf[off:off + n]
        assert (v.data_ptr() % 16 == 8) == bool(misalign)
        v.copy_(torch.from_numpy(h))
        dev.append(v)
    return host, dev


@pytest.mark.parametrize("misalign", [False, True])
@pytest.mark.parametrize("n", [1, 2, 7, 1000, 33_333, (1 << 20) + 3])
def test_stream_kernels_bitwise(n, misalign):
    from paper_2108_13622_b200 import _ops
    host, dev = _views(n, 4, n, misalign)
    cs = (1.0, 0.37, -2.5, 1e-3)
    for nt in (1, 2, 3, 4):
        ref = cs[0] * host[0]
        for k in range(1, nt):
            ref = ref + cs[k] * host[k]
        out, nrm, bad = _ops.lincomb(cs[:nt], dev[:nt], want_norm=True)
        assert np.array_equal(out.cpu().numpy(), ref)
        assert not bad
        # the flagged combination's norm is the norm kernel's, bit for bit
        assert nrm == _ops.norm(out)
        assert np.array_equal(_ops.lincomb(cs[:nt], dev[:nt]).cpu().numpy(), ref)
    q, qn = _ops.divide(dev[0], 3.7, want_norm=True)
    assert np.array_equal(q.cpu().numpy(), host[0] / 3.7)
    assert qn == _ops.norm(q)
    d, s = _ops.diff_norms(dev[0], dev[1])
    assert d == _ops.norm(_ops.lincomb((1.0, -1.0), dev[:2]))
    assert s == _ops.norm(dev[1])
    assert abs(s - np.linalg.norm(host[1])) <= 1e-13 * s
    # stage vector + offset in one pass
    for nt in (2, 3, 4):
        c1 = (1.0,) + cs[1:nt]
        ref = host[0].copy()
        for k in range(1, nt):
            ref = ref + c1[k] * host[k]
        out, diff, dn = _ops.lincomb_diff(c1, dev[:nt])
        assert np.array_equal(out.cpu().numpy(), ref)
        assert np.array_equal(diff.cpu().numpy(), ref - host[0])
        assert dn == _ops.norm(diff)
    # several combinations of the same vectors in one pass
    rows = ((64.0, -8.0, 0.0), (-60.0, -(285.0 / 8.0), 125.0 / 8.0),
            (0.0, 18.0, -(250.0 / 81.0)), (0.0, -60.0, 500.0 / 27.0))
    for nout in (2, 3, 4):
        outs = _ops.lincomb_multi(rows[:nout], dev[:3])
        for row, o in zip(rows, outs):
            keep = [(c, h) for c, h in zip(row, host) if c != 0.0]
            ref = keep[0][0] * keep[0][1]
            for c, h in keep[1:]:
                ref = ref + c * h
            assert np.array_equal(o.cpu().numpy(), ref)


def test_reductions_do_not_depend_on_alignment():
    """Aligned and misaligned copies of the same data reduce to the same bits
    (one traversal order, 128- or 64-bit accesses)."""
    from paper_2108_13622_b200 import _ops
    n = 777_777
    h0, a = _views(n, 2, 5, False)
    h1, b = _views(n, 2, 5, True)
    assert np.array_equal(h0[0], h1[0])
    assert _ops.norm(a[0]) == _ops.norm(b[0])
    assert _ops.diff_norms(a[0], a[1]) == _ops.diff_norms(b[0], b[1])
    assert _ops.lincomb((2.0, 3.0), a, want_norm=True)[1] == _ops.lincomb((2.0, 3.0), b, want_norm=True)[1]


def _problem(n=24, seed=4, harris=False):
    import paper_2108_13622_b200 as xb
    from paper_2108_13622_b200 import scenarios as sc
    s = sc.harris_setup(n) if harris else sc.kh_setup(n)
    q = sc.initial_fields(s)
    q = q + 1e-3 * np.random.default_rng(seed).standard_normal(q.shape)
    st = xb.StateGrid(n, n, s.dx, s.dy, _dev(q))
    op = xb.RhsOperator(xb.MhdRhs(st, xb.MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa)))
    return xb, st, op


@contextlib.contextmanager
def sync_per_term(fuse=True, zero_copy=True, adaptive=True):
    """Synchronous steps with one launch per Newton term (the large-grid path),
    on whatever grid the test uses."""
    from paper_2108_13622_b200 import integrators, leja, mhd
    old = (integrators.ASYNC, integrators.FUSE_STAGES, leja.LOOP_MAX_CELLS, leja.ZERO_COPY,
           leja.ADAPTIVE)
    integrators.ASYNC = False
    integrators.FUSE_STAGES = fuse
    leja.LOOP_MAX_CELLS = 0
    leja.ZERO_COPY = zero_copy
    leja.ADAPTIVE = adaptive
    for c in mhd._ctx_cache.values():
        c.loop_ok = None
    try:
        yield
    finally:
        (integrators.ASYNC, integrators.FUSE_STAGES, leja.LOOP_MAX_CELLS,
         leja.ZERO_COPY, leja.ADAPTIVE) = old
        for c in mhd._ctx_cache.values():
            c.loop_ok = None


@pytest.mark.parametrize("scheme,harris", [("EXPRB43", False), ("EXPRB54S4", True),
                                           ("EXPRB54S4", False)])
def test_fused_stage_algebra_is_bitwise(scheme, harris):
    """lincomb_diff + the JVP epilogue's (F(stage) - F(u)) - J d + the shared
    w_k pass against one kernel per reference expression, and the zero-copy
    Leja calls against the copying ones: same state, error estimate, counters."""
    from paper_2108_13622_b200 import leja
    xb, st, op = _problem(n=40 if harris else 24, harris=harris)
    u = st.flat()
    with sync_per_term():
        lin = xb.FrozenLinearization(op, u)
        alpha = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0)).alpha
    dt = 6.0 / alpha
    res = {}
    for key, kw in (("plain", dict(fuse=False, zero_copy=False)),
                    ("fused", dict(fuse=True, zero_copy=False)),
                    ("both", dict(fuse=True, zero_copy=True))):
        with sync_per_term(**kw):
            leja._coeff_cache.clear()
            lin = xb.FrozenLinearization(op, u)
            c0 = op.calls
            r = xb.step(getattr(xb.Scheme, scheme), op, u, dt, alpha=alpha, tol=1e-7, lin=lin)
            res[key] = (r, op.calls - c0)
    (a, ca) = res["plain"]
    assert a.converged and a.phi_iterations > 10
    for key in ("fused", "both"):
        (b, cb) = res[key]
        assert (b.converged, b.rhs_calls, b.phi_iterations, b.phi_applications, cb) == \
            (a.converged, a.rhs_calls, a.phi_iterations, a.phi_applications, ca)
        assert b.error_estimate == a.error_estimate
        assert torch.equal(b.new_state, a.new_state)


@pytest.mark.parametrize("l", [1, 3])
def test_zero_copy_leja_calls_are_bitwise(l):
    """In-place start (v read where it lies, c0*v formed by the first reader)
    and result hand-off against the copying start / copy-out: calls ending on
    an even term (stored interpolant), on an odd term (pending c*y), across
    the 64 -> 128 chunk growth, and on a zero vector."""
    from paper_2108_13622_b200 import leja
    xb, st, op = _problem(n=40)
    u = st.flat()
    with sync_per_term():
        lin = xb.FrozenLinearization(op, u)
        alpha = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0)).alpha
    v = _dev(np.random.default_rng(9).standard_normal(u.numel()))
    v_keep = v.clone()
    parities = set()
    for adt, tol in ((0.5, 1e-6), (3.0, 1e-10), (3.0, 1e-9), (7.0, 1e-8), (80.0, 1e-10)):
        out = {}
        for zc in (False, True):
            with sync_per_term(zero_copy=zc):
                leja._coeff_cache.clear()
                c0 = op.calls
                r = xb.apply_phi_leja(l, xb.JacobianAction(lin), v, adt / alpha,
                                      xb.shift_and_scale(adt), tol)
                out[zc] = (r, op.calls - c0, [(k, c.size) for k, c in leja._coeff_cache.items()])
        (a, ca, ka), (b, cb, kb) = out[False], out[True]
        assert (a.iterations, a.converged, a.residual, ca, ka) == \
            (b.iterations, b.converged, b.residual, cb, kb)
        assert torch.equal(a.vector, b.vector)
        assert torch.equal(v, v_keep)          # the caller's vector is only read
        parities.add(a.iterations & 1)
    assert parities == {0, 1}
    zero = torch.zeros_like(v)
    for zc in (False, True):
        with sync_per_term(zero_copy=zc):
            r = xb.apply_phi_leja(l, xb.JacobianAction(lin), zero, 1.0 / alpha,
                                  xb.shift_and_scale(1.0), 1e-10)
            assert r.converged and r.iterations == 2
            assert not r.vector.any()


@pytest.mark.parametrize("l", [1, 4])
def test_adaptive_lookahead_is_bitwise(l):
    """Variant pairs near the expected end (an odd term that may be the last
    one stores p and resolves its own residual) against the plain parity
    schedule (the next launch resolves it): same vector, degree, residual,
    RHS count and coefficient cache, whatever the degree hint says -- no hint
    (pairs from term 1), an exact hint, a hint far too low and far too high --
    for calls ending on odd and on even terms, across the chunk growth."""
    from paper_2108_13622_b200 import leja
    xb, st, op = _problem(n=40)
    u = st.flat()
    with sync_per_term():
        lin = xb.FrozenLinearization(op, u)
        alpha = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0)).alpha
    v = _dev(np.random.default_rng(11).standard_normal(u.numel()))
    parities = set()
    for adt, tol in ((0.5, 1e-6), (3.0, 1e-10), (3.0, 1e-9), (7.0, 1e-8), (20.0, 1e-9),
                     (80.0, 1e-10)):
        sh = xb.shift_and_scale(adt)
        hkey = (l, int(round(4.0 * np.log2(sh.theta))))

        def call(adaptive, hint):
            with sync_per_term(adaptive=adaptive):
                leja._coeff_cache.clear()
                leja._degree_hint.pop(hkey, None)
                if hint is not None:
                    leja._degree_hint[hkey] = hint
                c0 = op.calls
                r = xb.apply_phi_leja(l, xb.JacobianAction(lin), v, adt / alpha, sh, tol)
                return (r, op.calls - c0, [(k, c.size) for k, c in leja._coeff_cache.items()])
        a, ca, ka = call(False, None)
        parities.add(a.iterations & 1)
        for hint in (None, a.iterations + 1, 2, a.iterations + 40):
            b, cb, kb = call(True, hint)
            assert (a.iterations, a.converged, a.residual, ca, ka) == \
                (b.iterations, b.converged, b.residual, cb, kb), (adt, tol, hint)
            assert torch.equal(a.vector, b.vector), (adt, tol, hint)
    assert parities == {0, 1}


def test_zero_copy_call_reports_a_nonfinite_rhs_like_the_copying_call():
    """A direction that makes F(u + eps*y) non-finite at the first term: the
    reference raises RhsBlowupError from inside the matvec (mhd.py:225-231);
    both starts rebuild the same failing state (y is still the caller's v)."""
    from paper_2108_13622_b200 import leja
    xb, st, op = _problem(n=24)
    u = st.flat()
    with sync_per_term():
        lin = xb.FrozenLinearization(op, u)
        alpha = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0)).alpha
    v = _dev(np.random.default_rng(9).standard_normal(u.numel()))
    v[5] = float("inf")      # ||v|| = inf: eps = 0 and u + eps*v has a NaN cell
    msgs = []
    for zc in (False, True):
        with sync_per_term(zero_copy=zc):
            leja._coeff_cache.clear()
            with pytest.raises(xb.RhsBlowupError) as err:
                xb.apply_phi_leja(1, xb.JacobianAction(lin), v, 1.0 / alpha,
                                  xb.shift_and_scale(1.0), 1e-10)
            msgs.append((str(err.value), err.value.cells))
    assert msgs[0] == msgs[1]


def test_staged_pageable_upload_is_exact():
    """xmhd_h2d_staged (pageable NumPy -> device through page-locked slots filled
    by the host thread pool): exact bytes for sizes around the slot and
    cache-line boundaries, from an unaligned source."""
    from paper_2108_13622_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(3)
    for n in (1, 7, (16 << 20) // 8, (16 << 20) // 8 + 1, 5_000_011):
        base = rng.standard_normal(n + 1)
        src = base[1:]                       # 8 bytes off the allocation's alignment
        dst = torch.empty(n, dtype=torch.float64, device="cuda")
        rc = lib.xmhd_h2d_staged(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src.ctypes.data),
                                 src.nbytes, _lib.current_stream_handle())
        assert rc == 0
        torch.cuda.synchronize()
        assert np.array_equal(dst.cpu().numpy(), src)
    assert lib.xmhd_h2d_threads() >= 1


def test_term_timing_brackets_the_term_launches():
    """xmhd_term_timing (bench.py's in-region roofline timer): the fused terms of
    host-paced calls are bracketed by CUDA events while it is on, the sum is
    read and reset when it is switched, and the calls' results do not change."""
    from paper_2108_13622_b200 import _lib, leja
    xb, st, op = _problem(n=48)
    u = st.flat()
    lib = _lib.load()
    with sync_per_term():
        lin = xb.FrozenLinearization(op, u)
        alpha = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0)).alpha
        mv = xb.JacobianAction(lin)
        v = _dev(np.random.default_rng(3).standard_normal(u.numel()))
        h = lin.mhd.ctx.bind_stream()

        def call():
            leja._coeff_cache.clear()
            dt = 8.0 / alpha
            return xb.apply_phi_leja(1, mv, v, dt, xb.shift_and_scale(alpha * dt), 1e-9)

        base = call()
        got = ctypes.c_double(-1.0)
        assert lib.xmhd_term_timing(h, -1, ctypes.byref(got)) == 0 and got.value == 0.0
        assert lib.xmhd_term_timing(h, 1, None) == 0
        timed = [call() for _ in range(3)]
        assert lib.xmhd_term_timing(h, -1, ctypes.byref(got)) == 0
        running = got.value
        assert lib.xmhd_term_timing(h, 0, ctypes.byref(got)) == 0
        assert got.value == running > 0.0
        # a plausible device time: microseconds to milliseconds per term on this grid
        per_term = got.value / sum(r.iterations for r in timed)
        assert 1e-3 < per_term < 5.0
        after = call()
        assert lib.xmhd_term_timing(h, -1, ctypes.byref(got)) == 0 and got.value == 0.0
    for r in timed + [after]:
        assert (r.iterations, r.converged) == (base.iterations, base.converged)
        assert torch.equal(r.vector, base.vector)
