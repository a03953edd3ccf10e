"""ctypes binding of the C-ABI in ``include/xmhd_b200.h`` (``_xmhd_b200.so``).

The product path has no CPU fallback: if the shared library or a CUDA device is
missing, every entry point raises ``NativeUnavailable`` loudly.
"""

import ctypes
import os
import threading

import numpy as np
import torch

from paper_2108_13622_b200 import build as _build

OK, NONFINITE, BADARG, CUDA_ERROR = 0, 1, 2, 3
BAD_CELLS_LEN = 25   # XMHD_BAD_CELLS_LEN: count + 8 (field, i, j) triples
BC_PERIODIC, BC_REFLECTING, BC_HALO = 0, 1, 2
(LEJA_RUNNING, LEJA_CONVERGED, LEJA_BLOWUP, LEJA_RHS_NONFINITE, LEJA_NEED_COEFFS,
 LEJA_EXHAUSTED, LEJA_PEER_TIMEOUT, LEJA_MODE_ERROR) = range(8)


class NativeUnavailable(RuntimeError):
    """The sm_100a library or the CUDA device is not available."""


class NativeError(RuntimeError):
    pass


class LejaState(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int), ("iterations", ctypes.c_int),
                ("rhs_calls", ctypes.c_int), ("m", ctypes.c_int),
                ("residual", ctypes.c_double), ("eps", ctypes.c_double),
                ("ynorm", ctypes.c_double)]


class StepRecord(ctypes.Structure):
    """xmhd_step_record: the record of one asynchronous step."""
    _fields_ = [("rhs_nonfinite", ctypes.c_int), ("jvp_calls", ctypes.c_int),
                ("nleja", ctypes.c_int), ("lin_nonfinite", ctypes.c_int),
                ("err_diff", ctypes.c_double), ("err_ref", ctypes.c_double),
                ("lc_norm", ctypes.c_double), ("lc_nonfinite", ctypes.c_double),
                ("leja", LejaState * 32)]


_P = ctypes.c_void_p
_D = ctypes.c_double
_I = ctypes.c_int
_L = ctypes.c_longlong
_PD = ctypes.POINTER(ctypes.c_double)
_PI = ctypes.POINTER(ctypes.c_int)

_SIGS = {
    "xmhd_create": (_I, [ctypes.POINTER(_P), _I, _I, _D, _D, _D, _D, _D, _D, _D, _I, _I, _P]),
    "xmhd_destroy": (_I, [_P]),
    "xmhd_set_stream": (_I, [_P, _P]),
    "xmhd_last_error": (ctypes.c_char_p, []),
    "xmhd_plan_info": (_I, [_P, _PI]),
    "xmhd_launch_count": (_L, [_P]),
    "xmhd_set_halo": (_I, [_P, _P, _P, _P, _P]),
    "xmhd_rhs": (_I, [_P, _P, _P, _PI]),
    "xmhd_jvp": (_I, [_P, _P, _P, _D, _P, _P, _PI, _PD, _PI]),
    "xmhd_leja": (_I, [_P, _I, _P, _P, _D, _P, _D, _D, _D, _D, _PD, _PD, _I, _P, _PI, _PI,
                       _PD, _PI, _PI]),
    "xmhd_newton_coeffs": (_I, [_I, _D, _D, _PD, _I, _PD]),
    "xmhd_leja_schedule": (_I, [_I, _D, _D, _PD, _PD]),
    "xmhd_async_begin": (_I, [_P]),
    "xmhd_rhs_async": (_I, [_P, _P, _P]),
    "xmhd_jvp_async": (_I, [_P, _P, _P, _D, _P, _P]),
    "xmhd_leja_loop": (_I, [_P]),
    "xmhd_leja_loop_available": (_I, [_P]),
    "xmhd_set_loop_kind": (_I, [_P, _I]),
    "xmhd_set_leja_defer": (_I, [_P, _I]),
    "xmhd_leja_finish_async": (_I, [_P, _P]),
    "xmhd_lincomb_async": (_I, [_P, _P, _L, ctypes.POINTER(_P), _PD, _I]),
    "xmhd_diff_norms_async": (_I, [_P, _P, _P, _L]),
    "xmhd_async_fetch": (_I, [_P, ctypes.POINTER(StepRecord)]),
    "xmhd_step_async": (_I, [_P, _I, _P, _P, _D, _L, _D, _PD, _PD, _I, _D, _PD, _P, _P]),
    "xmhd_power": (_I, [_P, _P, _P, _D, _P, _P, _P, _I, _D, _PD, _PI, _PI, _PI]),
    "xmhd_linearize": (_I, [_P, _P, _P, _PD]),
    "xmhd_linearize_async": (_I, [_P, _P, _P]),
    "xmhd_linearize_check": (_I, [_P, _PI]),
    "xmhd_divb_async": (_I, [_P, _P, _P]),
    "xmhd_norm": (_I, [_P, _P, _L, _PD]),
    "xmhd_lincomb": (_I, [_P, _P, _L, ctypes.POINTER(_P), _PD, _I, _PD, _PI]),
    "xmhd_divide": (_I, [_P, _P, _P, _D, _L, _PD]),
    "xmhd_diff_norms": (_I, [_P, _P, _P, _L, _PD]),
    "xmhd_divb": (_I, [_P, _P, _P, _PD]),
    "xmhd_field_sums": (_I, [_P, _P, _PD]),
    "xmhd_cfl_speeds": (_I, [_P, _P, _PD]),
    "xmhd_leja_start": (_I, [_P, _P, _P, _D, _P, _D, _D, _D, _D, _PD, _PD, _I,
                             ctypes.POINTER(LejaState)]),
    "xmhd_leja_resume": (_I, [_P, _PD, _I, ctypes.POINTER(LejaState)]),
    "xmhd_leja_hint": (_I, [_P, _I]),
    "xmhd_leja_result": (_I, [_P, _P]),
    "xmhd_leja_current_y": (_I, [_P, _P]),
    "xmhd_leja_generic_start": (_I, [_P, _P, _L, _D, _D, _D, _D, _PD, _PD, _I,
                                     ctypes.POINTER(LejaState)]),
    "xmhd_leja_generic_step": (_I, [_P, _P, ctypes.POINTER(LejaState)]),
    "xmhd_leja_generic_resume": (_I, [_P, _PD, _I, ctypes.POINTER(LejaState)]),
    "xmhd_leja_generic_result": (_I, [_P, _P]),
    "xmhd_sumsq": (_I, [_P, _P, _L, _PD]),
    "xmhd_jvp_eps": (_I, [_P, _P, _P, _P, _D, _P, _PD]),
    "xmhd_leja_strip_start": (_I, [_P, _P, _P, _D, _P, _D, _D, _D, _D, _PD, _PD, _I, _P]),
    "xmhd_leja_strip_start_finalize": (_I, [_P, _P]),
    "xmhd_leja_strip_pack": (_I, [_P, _P, _P, _P, _P, _I, _I]),
    "xmhd_leja_strip_iterate": (_I, [_P, _P]),
    "xmhd_leja_strip_finalize": (_I, [_P, _P]),
    "xmhd_leja_query": (_I, [_P, ctypes.POINTER(LejaState)]),
    "xmhd_leja_set_coeffs": (_I, [_P, _PD, _I]),
    "xmhd_time_stencil": (_I, [_P, _I, _P, _P, _D, _P, _P, _I, _PD]),
    "xmhd_time_leja_iterations": (_I, [_P, _P, _P, _D, _P, _D, _D, _D, _PD, _PD, _I, _PD,
                                       _PD]),
    "xmhd_phi_divided_diffs": (_I, [_I, _PD, _I, _D, _PD]),
    "xmhd_krylov_mgs": (_I, [_P, ctypes.POINTER(_P), _I, _P, _L, _PD, _PD]),
    "xmhd_mgs_update": (_I, [_P, _P, _L, _P, _D, _P, _PD]),
    "xmhd_krylov_combine": (_I, [_P, ctypes.POINTER(_P), _PD, _I, _D, _L, _P]),
    "xmhd_leja_start_async": (_I, [_P, _P, _P, _D, _P, _D, _D, _D, _D, _PD, _PD, _I]),
    "xmhd_leja_launch": (_I, [_P, _I, _I]),
    "xmhd_leja_extend": (_I, [_P, _PD, _I, _I]),
    "xmhd_leja_sync": (_I, [_P, ctypes.POINTER(LejaState)]),
    "xmhd_p2p_alloc": (_I, [_P, _P]),
    "xmhd_p2p_connect": (_I, [_P, _I, _I, _P, _I]),
    "xmhd_p2p_connect_local": (_I, [ctypes.POINTER(_P), _I, _I]),
    "xmhd_p2p_probe": (_I, [_P, _D]),
    "xmhd_p2p_read_board": (_I, [_P, _PD]),
    "xmhd_leja_p2p_start": (_I, [_P, _P, _P, _D, _P, _D, _D, _D, _D, _PD, _PD, _I]),
    "xmhd_leja_p2p_run": (_I, [_P, ctypes.POINTER(LejaState)]),
    "xmhd_leja_p2p_emul_start": (_I, [ctypes.POINTER(_P), _I, ctypes.POINTER(_P),
                                      ctypes.POINTER(_P), _D, ctypes.POINTER(_P), _D, _D, _D,
                                      _D, _PD, _PD, _I]),
    "xmhd_leja_p2p_emul_run": (_I, [ctypes.POINTER(_P), _I, ctypes.POINTER(LejaState)]),
    "xmhd_leja_start_inplace": (_I, [_P, _P, _P, _D, _P, _D, _D, _D, _D, _PD, _PD, _I]),
    "xmhd_leja_set_dual_from": (_I, [_P, _I]),
    "xmhd_leja_set_pbuf": (_I, [_P, _P, _P]),
    "xmhd_leja_result_inplace": (_I, [_P, _PI]),
    "xmhd_stage_difference": (_I, [_P, _P, _P, _D, _P, _D, _P, _P, _PI, _PI]),
    "xmhd_lincomb_diff": (_I, [_P, _P, _P, _L, ctypes.POINTER(_P), _PD, _I, _PD]),
    "xmhd_lincomb_multi": (_I, [_P, ctypes.POINTER(_P), _I, _L, ctypes.POINTER(_P), _PD]),
    "xmhd_final_pair": (_I, [_P, _I, _P, _L, ctypes.POINTER(_P), _PD, _PD, _PI]),
    "xmhd_h2d_staged": (_I, [_P, _P, _L, _P]),
    "xmhd_h2d_threads": (_I, []),
    "xmhd_term_timing": (_I, [_P, _I, _PD]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def library_path():
    """The in-tree library; XMHD_SO points at an alternative build (A/B benchmarks)."""
    return os.environ.get("XMHD_SO") or _build.SO_PATH


def load(build_if_missing=True):
    """Load (building in-tree first if needed) and type the shared library."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = library_path()
        if build_if_missing and not os.environ.get("XMHD_SO"):
            try:
                _build.build_so()
            except (OSError, RuntimeError) as exc:
                if not os.path.exists(path):
                    raise NativeUnavailable(f"cannot build {path}: {exc}") from exc
        if not os.path.exists(path):
            raise NativeUnavailable(f"missing native library {path}; run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def require_cuda():
    if not torch.cuda.is_available():
        raise NativeUnavailable("the B200 hot path needs a CUDA device; none is visible "
                                "(no CPU fallback by design)")


def err_text():
    return load().xmhd_last_error().decode(errors="replace")


def check(rc, what):
    if rc == OK:
        return rc
    if rc == NONFINITE:
        return rc
    raise NativeError(f"{what} failed ({rc}): {err_text()}")


def ptr(t):
    """Device address of a contiguous CUDA float64 tensor."""
    if t is None:
        return None
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError("expected a contiguous CUDA float64 tensor")
    return ctypes.c_void_p(t.data_ptr())


def host_doubles(arr):
    a = np.ascontiguousarray(arr, dtype=np.float64)
    return a, a.ctypes.data_as(_PD)


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def current_stream_handle():
    """cudaStream_t of torch's current stream on the current device (the raw
    accessor skips the Stream object: this runs once per native call)."""
    if _raw_stream is not None:
        return ctypes.c_void_p(_raw_stream(torch.cuda.current_device()))
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class Context:
    """Owner of one native ``xmhd_ctx`` (a grid + physics parameter set)."""

    def __init__(self, nx, ny, dx, dy, mu, eta, kappa, gamma, mu0, bc_x, bc_y):
        require_cuda()
        self.lib = load()
        self.nx, self.ny = int(nx), int(ny)
        self.n = 8 * self.nx * self.ny
        h = ctypes.c_void_p()
        torch.cuda.init()
        rc = self.lib.xmhd_create(ctypes.byref(h), self.nx, self.ny, float(dx), float(dy),
                                  float(mu), float(eta), float(kappa), float(gamma),
                                  float(mu0), int(bc_x), int(bc_y), current_stream_handle())
        check(rc, "xmhd_create")
        self.h = h

    def bind_stream(self):
        st = current_stream_handle()
        if st.value != getattr(self, "_stream", -1):
            self.lib.xmhd_set_stream(self.h, st)
            self._stream = st.value
        return self.h

    def plan(self):
        out = (ctypes.c_int * 4)()
        check(self.lib.xmhd_plan_info(self.h, out), "xmhd_plan_info")
        return dict(units_x=out[0], units=out[1], seg_rows=out[2], grid=out[3])

    def launches(self):
        return int(self.lib.xmhd_launch_count(self.h))

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                self.lib.xmhd_destroy(h)
            except Exception:
                pass
            self.h = None
