"""Device vector primitives over the C-ABI (norms, linear combinations, division).

All vectors are contiguous CUDA float64 tensors.  Element-wise results follow
the reference's NumPy operation order exactly; norms are deterministic device
reductions.
"""

import ctypes
import math
import os
import threading

import numpy as np
import torch

from paper_2108_13622_b200 import _lib

_util = {}
_util_lock = threading.Lock()


_util_tls = threading.local()


def util_ctx():
    """A geometry-free context used for reductions on arbitrary vectors.

    One per (device, host thread): its reduction scratch must not be shared by
    concurrently enqueued work.
    """
    dev = torch.cuda.current_device()
    mine = getattr(_util_tls, "ctx", None)
    if mine is not None and mine[0] == dev:
        return mine[1]
    key = (dev, threading.get_ident())
    with _util_lock:
        c = _util.get(key)
        if c is None:
            c = _lib.Context(2, 2, 1.0, 1.0, 0.0, 0.0, 0.0, 5.0 / 3.0, 1.0,
                             _lib.BC_PERIODIC, _lib.BC_PERIODIC)
            _util[key] = c
    _util_tls.ctx = (dev, c)
    return c


def is_host(x):
    return isinstance(x, np.ndarray) or (torch.is_tensor(x) and not x.is_cuda) or \
        isinstance(x, (list, tuple, float, int))


class _Staging:
    """Pageable host -> device copies through page-locked chunks.

    A plain copy from pageable memory runs at ~11 GB/s on the B200 boxes
    (the driver stages it through its own bounce buffer on one thread).  The
    native ``xmhd_h2d_staged`` (csrc/hostio.cpp) keeps a persistent pool of
    host threads filling page-locked slots with streaming stores while the
    copy engine drains the previous ones on the current stream.  The
    reference's callers hand the API plain NumPy arrays, so this is the H2D of
    bench.py's ``e2e``.  (XMHD_H2D_PY=1: the same pipeline issued from Python,
    28 GB/s; kept for A/B, scripts/probe_h2d.py.)"""

    CHUNK = 32 << 20          # bytes per slot (Python pipeline)
    SLOTS = 4
    MIN_BYTES = 16 << 20      # below this a plain copy is as fast

    def __init__(self):
        self.lock = threading.Lock()
        self.slots = None
        self.events = [None] * self.SLOTS
        self.pool = None
        self.threads = 1
        self.python = bool(int(os.environ.get("XMHD_H2D_PY", "0") or "0"))

    def _init(self):
        from concurrent.futures import ThreadPoolExecutor
        n = self.CHUNK // 8
        self.slots = [torch.empty(n, dtype=torch.float64, pin_memory=True)
                      for _ in range(self.SLOTS)]
        try:
            cores = len(os.sched_getaffinity(0))
        except AttributeError:   # pragma: no cover
            cores = os.cpu_count() or 1
        self.threads = max(1, min(8, cores // 2))
        self.pool = ThreadPoolExecutor(self.threads, thread_name_prefix="xmhd-h2d")

    def copy(self, a):
        out = torch.empty(a.size, dtype=torch.float64, device="cuda")
        if not self.python:
            flat = a.reshape(-1)
            rc = _lib.load().xmhd_h2d_staged(ctypes.c_void_p(out.data_ptr()),
                                             ctypes.c_void_p(flat.ctypes.data), flat.nbytes,
                                             _lib.current_stream_handle())
            _lib.check(rc, "xmhd_h2d_staged")
            return out
        with self.lock:
            if self.slots is None:
                self._init()
            stream = torch.cuda.current_stream()
            chunk = self.CHUNK // 8
            flat = a.reshape(-1)
            for k, i0 in enumerate(range(0, flat.size, chunk)):
                m = min(chunk, flat.size - i0)
                s = k % self.SLOTS
                if self.events[s] is not None:
                    self.events[s].synchronize()      # the slot's previous copy is done
                buf = self.slots[s].numpy()
                cut = np.linspace(0, m, self.threads + 1).astype(np.int64)
                list(self.pool.map(
                    lambda j: np.copyto(buf[cut[j]:cut[j + 1]], flat[i0 + cut[j]:i0 + cut[j + 1]]),
                    range(self.threads)))
                out[i0:i0 + m].copy_(self.slots[s][:m], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
                self.events[s] = ev
        return out


_staging = _Staging()


def as_device(x, copy=False):
    """Contiguous CUDA float64 tensor view/copy of x (numpy, list, or tensor)."""
    if torch.is_tensor(x):
        t = x
        if not t.is_cuda:
            t = t.to(dtype=torch.float64).contiguous()
            if not t.is_pinned() and t.numel() * 8 >= _Staging.MIN_BYTES:
                _lib.require_cuda()
                return _staging.copy(t.numpy()).reshape(t.shape)
            t = t.to("cuda", non_blocking=t.is_pinned())
            return t
        if t.dtype != torch.float64:
            t = t.to(torch.float64)
        t = t.contiguous()
        return t.clone() if copy else t
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    _lib.require_cuda()
    if a.nbytes >= _Staging.MIN_BYTES:
        return _staging.copy(a).reshape(a.shape)
    return torch.from_numpy(a).to("cuda")


def to_host(t):
    """D2H into page-locked memory (torch's caching host allocator) -> NumPy view.

    The returned array keeps its pinned block alive; the block returns to the
    pool when the array is released, so repeated calls do not re-pin memory.
    """
    t = t.detach()
    if not t.is_cuda:
        return t.numpy()
    host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    host.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return host.numpy()


def like(result, template):
    """Return `result` (device tensor) in the container type of `template`."""
    return to_host(result) if is_host(template) else result


def _h(ctx):
    return (ctx or util_ctx()).bind_stream()


# Cross-rank reducer of the y-strip decomposition (strips.Reducer); None = one
# domain.  Host-thread local, so ranks emulated by threads stay independent.
_tls = threading.local()


def set_reducer(reducer):
    """Install (or clear with None) the cross-rank reduction used by every norm."""
    prev = getattr(_tls, "reducer", None)
    _tls.reducer = reducer
    return prev


def reducer():
    return getattr(_tls, "reducer", None)


def sumsq(x, ctx=None):
    """Local sum of squares of a device vector (deterministic)."""
    lib = _lib.load()
    out = ctypes.c_double()
    _lib.check(lib.xmhd_sumsq(_h(ctx), _lib.ptr(x), x.numel(), ctypes.byref(out)), "xmhd_sumsq")
    return float(out.value)


def norm(x, ctx=None):
    """np.linalg.norm(x) of a device vector (global over ranks on y-strips)."""
    red = reducer()
    if red is not None:
        return math.sqrt(red.sum([sumsq(x, ctx)])[0])
    lib = _lib.load()
    out = ctypes.c_double()
    _lib.check(lib.xmhd_norm(_h(ctx), _lib.ptr(x), x.numel(), ctypes.byref(out)), "xmhd_norm")
    return float(out.value)


def global_max(values):
    red = reducer()
    return red.max(list(values)) if red is not None else list(values)


def global_sum(values):
    red = reducer()
    return red.sum(list(values)) if red is not None else list(values)


def lincomb(coeffs, vecs, out=None, want_norm=False, ctx=None):
    """((c0*v0 + c1*v1) + c2*v2) + c3*v3 with one rounding per operation.

    Returns out, or (out, norm, nonfinite) when want_norm.
    """
    assert 1 <= len(vecs) == len(coeffs) <= 4
    lib = _lib.load()
    n = vecs[0].numel()
    if out is None:
        out = torch.empty_like(vecs[0])
    arr = (ctypes.c_void_p * 4)(*[ctypes.c_void_p(v.data_ptr()) for v in vecs])
    cs = (ctypes.c_double * 4)(*[float(c) for c in coeffs])
    if want_norm:
        nrm = ctypes.c_double()
        bad = ctypes.c_int()
        rc = lib.xmhd_lincomb(_h(ctx), _lib.ptr(out), n, arr, cs, len(vecs), ctypes.byref(nrm),
                              ctypes.byref(bad))
        _lib.check(rc, "xmhd_lincomb")
        red = reducer()
        if red is not None:
            s, b = red.sum([nrm.value * nrm.value, float(bad.value)])
            return out, math.sqrt(s), b > 0.0
        return out, float(nrm.value), bool(bad.value)
    rc = lib.xmhd_lincomb(_h(ctx), _lib.ptr(out), n, arr, cs, len(vecs), None, None)
    _lib.check(rc, "xmhd_lincomb")
    return out


def lincomb_diff(coeffs, vecs, ctx=None):
    """(out, out - vecs[0], ||out - vecs[0]||) in one pass: a stage vector
    u + sum c_k p_k and the direction stage - u of its stage difference
    (integrators.py:139-153).  Single domain only (the norm is local)."""
    assert 2 <= len(vecs) == len(coeffs) <= 4 and reducer() is None
    lib = _lib.load()
    out = torch.empty_like(vecs[0])
    diff = torch.empty_like(vecs[0])
    arr = (ctypes.c_void_p * 4)(*[ctypes.c_void_p(v.data_ptr()) for v in vecs])
    cs = (ctypes.c_double * 4)(*[float(c) for c in coeffs])
    nrm = ctypes.c_double()
    rc = lib.xmhd_lincomb_diff(_h(ctx), _lib.ptr(out), _lib.ptr(diff), out.numel(), arr, cs,
                               len(vecs), ctypes.byref(nrm))
    _lib.check(rc, "xmhd_lincomb_diff")
    return out, diff, float(nrm.value)


def lincomb_multi(rows, vecs, ctx=None):
    """[sum_k rows[j][k] * vecs[k] for j] (k in order, zero coefficients skipped)
    for 2-4 combinations of the same three vectors, in one pass."""
    assert len(vecs) == 3 and 2 <= len(rows) <= 4
    lib = _lib.load()
    outs = [torch.empty_like(vecs[0]) for _ in rows]
    oarr = (ctypes.c_void_p * 4)(*[ctypes.c_void_p(o.data_ptr()) for o in outs])
    varr = (ctypes.c_void_p * 3)(*[ctypes.c_void_p(v.data_ptr()) for v in vecs])
    flat = [float(c) for row in rows for c in row]
    cs = (ctypes.c_double * 12)(*(flat + [0.0] * (12 - len(flat))))
    rc = lib.xmhd_lincomb_multi(_h(ctx), oarr, len(rows), vecs[0].numel(), varr, cs)
    _lib.check(rc, "xmhd_lincomb_multi")
    return outs


def final_pair(scheme_code, coeffs, vecs, ctx=None):
    """(hi, ||lo - hi||, ||hi||, nonfinite) of a step's two embedded solutions in
    one pass (csrc/vec.cu FinalPairOp; scheme_code 0 = EXPRB43 with 4 vectors,
    1 = EXPRB54s4 with 6).  Single domain only (the norms are local)."""
    assert reducer() is None and len(vecs) == len(coeffs) == (4 if scheme_code == 0 else 6)
    lib = _lib.load()
    out = torch.empty_like(vecs[0])
    arr = (ctypes.c_void_p * 6)(*[ctypes.c_void_p(v.data_ptr()) for v in vecs])
    cs = (ctypes.c_double * 6)(*[float(c) for c in coeffs])
    err = (ctypes.c_double * 2)()
    bad = ctypes.c_int()
    rc = lib.xmhd_final_pair(_h(ctx), int(scheme_code), _lib.ptr(out), out.numel(), arr, cs, err,
                             ctypes.byref(bad))
    _lib.check(rc, "xmhd_final_pair")
    return out, float(err[0]), float(err[1]), bool(bad.value)


def divide(x, d, out=None, want_norm=False, ctx=None):
    """x / d element-wise (IEEE); optionally also ||x / d||."""
    lib = _lib.load()
    if out is None:
        out = torch.empty_like(x)
    if want_norm:
        nrm = ctypes.c_double()
        rc = lib.xmhd_divide(_h(ctx), _lib.ptr(out), _lib.ptr(x), float(d), x.numel(),
                             ctypes.byref(nrm))
        _lib.check(rc, "xmhd_divide")
        return out, float(nrm.value)
    rc = lib.xmhd_divide(_h(ctx), _lib.ptr(out), _lib.ptr(x), float(d), x.numel(), None)
    _lib.check(rc, "xmhd_divide")
    return out


def diff_norms(a, b, ctx=None):
    """(||a - b||, ||b||) of two device vectors (global over ranks on y-strips)."""
    red = reducer()
    if red is not None:
        d = lincomb((1.0, -1.0), (a, b), ctx=ctx)
        s_d, s_b = red.sum([sumsq(d, ctx), sumsq(b, ctx)])
        return math.sqrt(s_d), math.sqrt(s_b)
    lib = _lib.load()
    out = (ctypes.c_double * 2)()
    rc = lib.xmhd_diff_norms(_h(ctx), _lib.ptr(a), _lib.ptr(b), a.numel(), out)
    _lib.check(rc, "xmhd_diff_norms")
    return float(out[0]), float(out[1])
