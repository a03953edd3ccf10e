"""Real Leja points and phi-function actions by Newton interpolation on the B200.

Host mirror of the reference module ``pkg/src/xmhd/leja.py`` (same names,
signatures, result type and non-convergence-as-a-flag behaviour).

When the matvec is the frozen MHD Jacobian (``JacobianAction`` over a device
``RhsOperator(MhdRhs)``), the whole Newton recurrence runs device-side: every
term is one fused stencil launch that forms F(u + eps*y), the FD Jacobian
action, the next basis vector, the interpolant update and both norms, and the
last CTA updates the convergence control in device memory (csrc/stencil.cu).
The host only intervenes when the coefficient chunk must grow
(leja.py:128-130), keeping the reference's coefficient cache semantics.

Any other matvec callable runs the same recurrence with the vector update in
a device kernel around the caller's matvec.
"""

import ctypes
import os
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np
import torch

from paper_2108_13622_b200 import _lib
from paper_2108_13622_b200 import _ops
from paper_2108_13622_b200.phi import _check_order, _phi_divided_diffs

LEJA_MAX = 500       # leja.py:15
_GRID_SIZE = 10001   # leja.py:18

_sequence_cache = None
_coeff_cache = {}
_tls = threading.local()


def _cache():
    """The coefficient cache of this host thread (the main thread's is _coeff_cache).

    One process per GPU uses only the main thread's cache; ranks emulated by
    threads (tests) get independent caches like independent processes would.
    """
    if threading.current_thread() is threading.main_thread():
        return _coeff_cache
    c = getattr(_tls, "cache", None)
    if c is None:
        c = _tls.cache = {}
    return c


def _greedy_leja(count):
    """Sequential argmax of the log-distance product over a uniform grid (leja.py:24-37)."""
    cand = np.linspace(-2.0, 2.0, _GRID_SIZE)
    out = np.empty(count)
    out[0] = 2.0
    with np.errstate(divide="ignore"):
        score = np.log(np.abs(cand - out[0]))
        for k in range(1, count):
            top = score.max()
            # symmetric ties resolve toward the positive candidate
            near = np.nonzero(score >= top - 1e-12 * max(1.0, abs(top)))[0]
            out[k] = cand[near[np.argmax(cand[near])]]
            score += np.log(np.abs(cand - out[k]))
    return out


def leja_points(count=LEJA_MAX):
    """The first `count` Leja points of [-2, 2], starting from 2 (leja.py:40-53)."""
    global _sequence_cache
    if not 1 <= count <= LEJA_MAX:
        raise ValueError(f"count must lie in [1, {LEJA_MAX}], got {count}")
    if _sequence_cache is None:
        seq = _greedy_leja(LEJA_MAX)
        seq.setflags(write=False)
        _sequence_cache = seq
    return _sequence_cache[:count]


@dataclass(frozen=True)
class ShiftScale:
    """Affine map placing the spectral interval [-alpha, 0] onto [-2, 2] (leja.py:56-60)."""
    q: float
    theta: float


def shift_and_scale(alpha):
    """q = -alpha/2, theta = alpha/4 (leja.py:63-72)."""
    if alpha <= 0:
        raise ValueError("spectral magnitude must be positive; "
                         "callers handle the degenerate spectrum separately")
    return ShiftScale(q=-0.5 * alpha, theta=0.25 * alpha)


@dataclass
class PhiApplyResult:
    """Outcome of one iterative phi-function action (leja.py:75-81)."""
    vector: object
    iterations: int
    converged: bool
    residual: float


def _compute_coeffs(l, q, theta, count):
    xi = leja_points(LEJA_MAX)[:count]
    return _phi_divided_diffs(l, q + theta * xi, subdiag=theta) / theta ** l


# Speculative chunk growth: while the device runs the Newton terms of the
# current chunk, a host thread computes the next chunk (a pure function of
# (l, q, theta, count), so the values are the ones an on-demand computation
# would produce).  The cache below still follows the reference's policy.
_spec_pool = ThreadPoolExecutor(max_workers=4, thread_name_prefix="leja-coeffs")
_spec_all = {}


class _SpecView:
    """Per-host-thread view of the speculation table (like _cache()): ranks
    emulated by threads share (l, q, theta, count) keys and must not pop or
    iterate each other's entries."""

    def _d(self):
        if threading.current_thread() is threading.main_thread():
            return _spec_all
        d = getattr(_tls, "spec", None)
        if d is None:
            d = _tls.spec = {}
        return d

    def __contains__(self, key):
        return key in self._d()

    def __iter__(self):
        return iter(list(self._d()))

    def __setitem__(self, key, value):
        self._d()[key] = value

    def pop(self, key, default=None):
        return self._d().pop(key, default)


_spec = _SpecView()
_degree_hint = {}


def _speculate(l, q, theta, count):
    hit = _cache().get((l, q, theta))
    if (hit is not None and hit.size >= count) or (l, q, theta, count) in _spec:
        return
    _spec[(l, q, theta, count)] = _spec_pool.submit(_compute_coeffs, l, q, theta, count)


def _drop_speculation(l, q, theta):
    for key in [k for k in _spec if k[:3] == (l, q, theta)]:
        fut = _spec.pop(key, None)
        if fut is not None:
            fut.cancel()


def _newton_coeffs(l, q, theta, count):
    """Divided differences of xi -> phi_l(q + theta*xi) at the Leja points, / theta**l.

    Cached per exact (l, q, theta) with the reference's FIFO policy
    (leja.py:84-100); the heavy part runs in the native C++ port.
    """
    key = (l, q, theta)
    cache = _cache()
    hit = cache.get(key)
    if hit is not None and hit.size >= count:
        return hit
    fut = _spec.pop((l, q, theta, count), None)
    if fut is not None and (fut.running() or fut.done()):
        coeffs = fut.result()
    else:
        if fut is not None:
            fut.cancel()
        coeffs = _compute_coeffs(l, q, theta, count)
    if len(cache) > 64:
        cache.pop(next(iter(cache)))
    cache[key] = coeffs
    return coeffs


def newton_coeffs_many(keys, count=64):
    """_newton_coeffs for a sequence of (l, q, theta) in call order, the cache
    misses computed concurrently on the coefficient pool (the divided
    differences release the GIL); the cache sees the same lookups and inserts,
    in the same order, as one _newton_coeffs call per key."""
    cache = _cache()
    futs = {}
    for key in keys:
        hit = cache.get(key)
        if (hit is None or hit.size < count) and key not in futs:
            spec = _spec.pop(key + (count,), None)
            futs[key] = spec if spec is not None else _spec_pool.submit(_compute_coeffs, *key,
                                                                        count)
    out = []
    for key in keys:
        hit = cache.get(key)
        if hit is not None and hit.size >= count:
            out.append(hit)
            continue
        fut = futs.pop(key, None)
        coeffs = fut.result() if fut is not None else _compute_coeffs(*key, count)
        if len(cache) > 64:
            cache.pop(next(iter(cache)))
        cache[key] = coeffs
        out.append(coeffs)
    return out


class JacobianAction:
    """The matvec w -> jvp(lin, w) of a frozen linearization.

    ``_PhiBroker`` hands this object to ``apply_phi_leja``; when the
    linearization wraps the device MHD operator the Leja loop is fused.
    """

    def __init__(self, lin):
        self.lin = lin

    @property
    def fused(self):
        return self.lin.mhd is not None

    def __call__(self, w):
        from paper_2108_13622_b200.linearize import jvp
        return jvp(self.lin, w)


def _grow(l, q, theta, chunk, coeffs, m):
    """Coefficient growth at m >= coeffs.size exactly as leja.py:128-130."""
    chunk = min(2 * chunk, LEJA_MAX)
    coeffs = _newton_coeffs(l, q, theta, chunk)
    if m >= coeffs.size:
        # the reference indexes coeffs[m] next and fails the same way
        raise IndexError(f"index {m} is out of bounds for axis 0 with size {coeffs.size}")
    return chunk, coeffs


def _grow_pending(l, q, theta, chunk, m):
    """The table leja.py:128-130 fetches at term m, WITHOUT touching the cache.

    A device loop with the lookahead schedule can stop for coefficients at an
    odd term whose convergence is not resolved yet; if the call turns out to
    have converged on the term before, the reference never grew the table.
    So the grown table is only uploaded here, and ``_commit_growth`` performs
    the cache insert afterwards for the boundaries the call actually crossed.
    Returns (chunk, table, computed): ``computed`` is False when the reference
    would have found the table in the cache (no insert then)."""
    chunk = min(2 * chunk, LEJA_MAX)
    hit = _cache().get((l, q, theta))
    if hit is not None and hit.size >= chunk:
        table, computed = hit, False
    else:
        fut = _spec.pop((l, q, theta, chunk), None)
        table = fut.result() if fut is not None else _compute_coeffs(l, q, theta, chunk)
        computed = True
    if m >= table.size:
        raise IndexError(f"index {m} is out of bounds for axis 0 with size {table.size}")
    return chunk, table, computed


def _commit_growth(l, q, theta, grown, iterations):
    """Cache inserts of the growths in ``grown`` ([(m, table, computed)]) whose
    term m the call reached (iterations >= m), in order."""
    for m_b, table, computed in grown:
        if computed and iterations >= m_b:
            _cache_insert(l, q, theta, table)


def _ptr_d(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _growth_plan(size, chunk=64):
    """[(m, chunk)]: the chunk the reference fetches when the term index m reaches
    the end of its coefficient table (leja.py:128-130), in order.  Stops where
    the reference would index past the table (a cached table larger than the
    doubled chunk is returned unchanged): the device then stops at that m."""
    plan = []
    while size < LEJA_MAX:
        chunk = min(2 * chunk, LEJA_MAX)
        if chunk <= size:
            break
        plan.append((size, chunk))
        size = chunk
    return plan


def _cache_insert(l, q, theta, coeffs):
    """The cache update _newton_coeffs performs on a miss (leja.py:96-99)."""
    cache = _cache()
    if len(cache) > 64:
        cache.pop(next(iter(cache)))
    cache[(l, q, theta)] = coeffs


def drive_fused(lib, h, l, q, theta, coeffs, peer=False):
    """Host-paced device Leja loop shared by the single-GPU and y-strip drivers.

    Enqueues iteration kernels in batches sized by the degree of earlier calls
    at a similar interval, and extends the device coefficient table ahead of
    the term that first needs a grown chunk: the chunk is computed on a host
    thread while the device iterates and its new entries are uploaded in
    stream order (xmhd_leja_extend), so the loop never waits for the host at a
    chunk boundary.  The reference's cache growth is replayed afterwards for
    the boundaries the iteration actually crossed.  Returns the final state.
    """
    plan = _growth_plan(coeffs.size)
    futs = {}

    def fut(k):
        if k < len(plan) and k not in futs:
            futs[k] = _spec_pool.submit(_compute_coeffs, l, q, theta, plan[k][1])
        return futs.get(k)

    hkey = (l, int(round(4.0 * np.log2(theta))) if theta > 0 else 0)
    batch = max(2, int(_degree_hint.get(hkey, 2)))
    if not peer:
        # variant pairs from a few terms before the expected end (csrc/kernels.h,
        # leja_next_pmode): a call ending on an odd term costs no extra launch
        _lib.check(lib.xmhd_leja_set_dual_from(h, max(1, batch - 6) if ADAPTIVE else 0),
                   "xmhd_leja_set_dual_from")
    # every chunk the expected degree will reach is computed from the start, in
    # parallel (the divided differences release the GIL), so a slow host core
    # never makes the device wait at a chunk boundary
    fut(0)
    for kk in range(1, len(plan)):
        if plan[kk][0] <= batch + batch // 4 + 8:
            fut(kk)
    table_end, k, enq = coeffs.size, 0, 0
    grown = []
    st = _lib.LejaState()
    target = batch
    try:
        while True:
            while enq < min(target, LEJA_MAX - 1):
                if k < len(plan) and enq + 1 >= plan[k][0]:
                    arr = np.ascontiguousarray(fut(k).result())
                    fut(k + 1)
                    _lib.check(lib.xmhd_leja_extend(h, _ptr_d(arr), table_end, plan[k][1]),
                               "xmhd_leja_extend")
                    grown.append(arr)
                    table_end = plan[k][1]
                    k += 1
                    continue
                stop = min(target, LEJA_MAX - 1)
                if k < len(plan):
                    stop = min(stop, plan[k][0] - 1)
                _lib.check(lib.xmhd_leja_launch(h, stop - enq, int(peer)), "xmhd_leja_launch")
                enq = stop
            _lib.check(lib.xmhd_leja_sync(h, ctypes.byref(st)), "xmhd_leja_sync")
            # a batch that ended exactly at a chunk boundary leaves the device
            # waiting for the extension the loop above enqueues next
            waiting = (st.status == _lib.LEJA_NEED_COEFFS and k < len(plan) and
                       st.m == plan[k][0])
            if st.status != _lib.LEJA_RUNNING and not waiting:
                break
            batch = min(2 * batch, 64)
            target = enq + batch
    finally:
        for f in futs.values():
            f.cancel()
    for (m_b, _), arr in zip(plan, grown):
        if st.iterations >= m_b:
            _cache_insert(l, q, theta, arr)
    if st.status == _lib.LEJA_NEED_COEFFS:
        # only where the reference itself fails (see _growth_plan)
        chunk = plan[-1][1] if plan else 64
        _grow(l, q, theta, chunk, _cache().get((l, q, theta)), st.m)
        raise RuntimeError("coefficient table ended early")   # not reached
    # + 1: on one domain a term's convergence is resolved by the next launch
    # (deferred interpolant with lookahead, csrc/kernels.h)
    _degree_hint[hkey] = int(st.iterations) + 1
    return st


def apply_phi_leja(l, matvec, v, dt, shift, tol):
    """Approximate phi_l(J dt) v with J available only through `matvec` (leja.py:103-150).

    Newton terms are added one at a time (one matvec each); converged after two
    consecutive increments below tol * max(1, ||result||); non-convergence
    (500-term cap, basis overflow) is reported in the result, not raised.
    """
    _check_order(l)
    if tol <= 0:
        raise ValueError("tolerance must be positive")
    xi = np.ascontiguousarray(leja_points(LEJA_MAX))
    if isinstance(matvec, JacobianAction) and matvec.fused:
        from paper_2108_13622_b200.strips import StripMhd, apply_phi_leja_strips
        if isinstance(matvec.lin.mhd, StripMhd):
            return apply_phi_leja_strips(l, matvec.lin, v, dt, shift, tol, xi)
        return _apply_fused(l, matvec.lin, v, dt, shift, tol, xi)
    return _apply_generic(l, matvec, v, dt, shift, tol, xi)


# Grids up to this many cells run the Leja loop as one cooperative launch per
# phi-action (xmhd_leja_loop); larger ones, where a term costs hundreds of
# microseconds, keep the host-paced batches of drive_fused (which also extend
# the coefficient table ahead of the device without stopping it).
LOOP_MAX_CELLS = int(os.environ.get("XMHD_LOOP_MAX_CELLS", str(1 << 20)))
# Host-paced calls start in place (no y = v copy, no p = c0*v pass) and hand
# the result back in one of two caller-owned interpolant buffers instead of
# copying it out; XMHD_ZERO_COPY=0 restores the copies (A/B, tests).
ZERO_COPY = bool(int(os.environ.get("XMHD_ZERO_COPY", "1") or "1"))
# Variant pairs near the expected end of a host-paced call (adaptive lookahead);
# XMHD_ADAPTIVE=0: the plain parity schedule (A/B, tests).
ADAPTIVE = bool(int(os.environ.get("XMHD_ADAPTIVE", "1") or "1"))


def loop_available(mhd):
    """True when phi-actions on this operator run as one device loop."""
    ctx = mhd.ctx
    ok = getattr(ctx, "loop_ok", None)
    if ok is None:
        ok = (ctx.nx * ctx.ny <= LOOP_MAX_CELLS and
              bool(_lib.load().xmhd_leja_loop_available(ctx.h)))
        ctx.loop_ok = ok
    return ok


def drive_loop(lib, h, l, q, theta, coeffs):
    """Device loop with the reference's chunk growth (leja.py:128-130) at the
    terms where the table ends: the loop stops with NEED_COEFFS, the grown
    chunk's new entries are appended, and the loop resumes."""
    st = _lib.LejaState()
    chunk = 64
    size = coeffs.size
    grown = []
    while True:
        _lib.check(lib.xmhd_leja_loop(h), "xmhd_leja_loop")
        _lib.check(lib.xmhd_leja_sync(h, ctypes.byref(st)), "xmhd_leja_sync")
        if st.status != _lib.LEJA_NEED_COEFFS:
            _commit_growth(l, q, theta, grown, st.iterations)
            return st
        m = int(st.m)
        chunk, table, computed = _grow_pending(l, q, theta, chunk, m)
        grown.append((m, table, computed))
        arr = np.ascontiguousarray(table)
        _lib.check(lib.xmhd_leja_extend(h, _ptr_d(arr), size, arr.size), "xmhd_leja_extend")
        size = arr.size


def _start(lib, h, l, lin, vd, dt, q, theta, tol, xi, coeffs, inplace=False):
    start = lib.xmhd_leja_start_inplace if inplace else lib.xmhd_leja_start_async
    rc = start(h, _lib.ptr(lin.base_state), _lib.ptr(lin.base_rhs), float(lin._base_norm),
               _lib.ptr(vd), float(dt), float(q), float(theta), float(tol), _ptr_d(xi),
               _ptr_d(coeffs), int(coeffs.size))
    _lib.check(rc, "xmhd_leja_start_async")


def apply_phi_async(l, lin, v, dt, shift, tol):
    """One phi-action enqueued without any host wait (asynchronous steps).

    Only the first coefficient chunk is on the device: a call that reaches its
    end stops with NEED_COEFFS, which the step's record reports and the caller
    answers by replaying the step synchronously.  Returns the device vector
    that receives the interpolant; its final state goes to the step record.
    """
    _check_order(l)
    q, theta = shift.q, shift.theta
    lib = _lib.load()
    xi = np.ascontiguousarray(leja_points(LEJA_MAX))
    vd = _ops.as_device(v).reshape(-1)
    coeffs = np.ascontiguousarray(_newton_coeffs(l, q, theta, 64))
    h = lin.mhd.ctx.bind_stream()
    _start(lib, h, l, lin, vd, dt, q, theta, tol, xi, coeffs)
    _lib.check(lib.xmhd_leja_loop(h), "xmhd_leja_loop")
    p = torch.empty_like(vd)
    _lib.check(lib.xmhd_leja_finish_async(h, _lib.ptr(p)), "xmhd_leja_finish_async")
    return p


def cache_snapshot():
    """Copy of the coefficient cache (restored when an asynchronous step is replayed)."""
    return dict(_cache())


def cache_restore(snap):
    cache = _cache()
    cache.clear()
    cache.update(snap)


def _apply_fused(l, lin, v, dt, shift, tol, xi):
    from paper_2108_13622_b200.linearize import RhsBlowupError
    q, theta = shift.q, shift.theta
    mhd = lin.mhd
    lib = _lib.load()
    vd = _ops.as_device(v).reshape(-1)
    coeffs = np.ascontiguousarray(_newton_coeffs(l, q, theta, 64))
    h = mhd.ctx.bind_stream()
    looped = loop_available(mhd)
    pair = None
    if not looped and ZERO_COPY:
        # host-paced terms (large grids): v is read in place and the interpolant
        # lives in two caller-owned buffers, one of which becomes the result
        pair = (torch.empty_like(vd), torch.empty_like(vd))
        _lib.check(lib.xmhd_leja_set_pbuf(h, _lib.ptr(pair[0]), _lib.ptr(pair[1])),
                   "xmhd_leja_set_pbuf")
    try:
        _start(lib, h, l, lin, vd, dt, q, theta, tol, xi, coeffs, inplace=pair is not None)
        if looped:
            st = drive_loop(lib, h, l, q, theta, coeffs)
        else:
            st = drive_fused(lib, h, l, q, theta, coeffs)
        if pair is not None and st.status != _lib.LEJA_RHS_NONFINITE:
            which = ctypes.c_int()
            _lib.check(lib.xmhd_leja_result_inplace(h, ctypes.byref(which)),
                       "xmhd_leja_result_inplace")
    finally:
        if pair is not None:
            lib.xmhd_leja_set_pbuf(h, None, None)
    lin.rhs.calls += st.rhs_calls
    if st.status == _lib.LEJA_RHS_NONFINITE:
        # the reference raises from inside the matvec (mhd.py:225-231); rebuild
        # the failing state u + eps*y to report the same cells
        y = torch.empty_like(vd)
        _lib.check(lib.xmhd_leja_current_y(h, _lib.ptr(y)), "xmhd_leja_current_y")
        x = _ops.lincomb((1.0, st.eps), (lin.base_state, y))
        try:
            mhd(x)
        except RhsBlowupError as err:
            raise err
        raise RhsBlowupError("non-finite rhs inside the fused Leja iteration")
    if pair is not None:
        p = pair[which.value]
    else:
        p = torch.empty_like(vd)
        _lib.check(lib.xmhd_leja_result(h, _lib.ptr(p)), "xmhd_leja_result")
    return PhiApplyResult(vector=_ops.like(p, v), iterations=int(st.iterations),
                          converged=st.status == _lib.LEJA_CONVERGED,
                          residual=float(st.residual))


def _apply_generic(l, matvec, v, dt, shift, tol, xi):
    q, theta = shift.q, shift.theta
    lib = _lib.load()
    host_io = _ops.is_host(v)
    vd = _ops.as_device(v, copy=True).reshape(-1)
    ctx = _ops.util_ctx()
    h = ctx.bind_stream()
    chunk = 64
    coeffs = np.ascontiguousarray(_newton_coeffs(l, q, theta, chunk))
    st = _lib.LejaState()
    rc = lib.xmhd_leja_generic_start(h, _lib.ptr(vd), vd.numel(), float(dt), float(q),
                                     float(theta), float(tol), _ptr_d(xi), _ptr_d(coeffs),
                                     int(coeffs.size), ctypes.byref(st))
    _lib.check(rc, "xmhd_leja_generic_start")
    y = torch.empty_like(vd)
    try:
        while st.status in (_lib.LEJA_RUNNING, _lib.LEJA_NEED_COEFFS):
            if st.status == _lib.LEJA_NEED_COEFFS:
                chunk, grown = _grow(l, q, theta, chunk, coeffs, st.m)
                coeffs = np.ascontiguousarray(grown)
                rc = lib.xmhd_leja_generic_resume(h, _ptr_d(coeffs), int(coeffs.size),
                                                  ctypes.byref(st))
                _lib.check(rc, "xmhd_leja_generic_resume")
                continue
            _lib.check(lib.xmhd_leja_current_y(h, _lib.ptr(y)), "xmhd_leja_current_y")
            w = matvec(_ops.to_host(y) if host_io else y)
            wd = _ops.as_device(w).reshape(-1)
            rc = lib.xmhd_leja_generic_step(h, _lib.ptr(wd), ctypes.byref(st))
            _lib.check(rc, "xmhd_leja_generic_step")
    finally:
        p = torch.empty_like(vd)
        _lib.check(lib.xmhd_leja_generic_result(h, _lib.ptr(p)), "xmhd_leja_generic_result")
    return PhiApplyResult(vector=_ops.like(p, v), iterations=int(st.iterations),
                          converged=st.status == _lib.LEJA_CONVERGED,
                          residual=float(st.residual))
