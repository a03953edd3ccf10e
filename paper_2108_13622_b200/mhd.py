"""Resistive-MHD state, parameters and right-hand side on the B200.

Host mirror of the reference module ``pkg/src/xmhd/mhd.py``: same names,
argument meaning, layout (8, ny, nx) and error behaviour (``RhsBlowupError``
listing up to 8 non-finite cells in C order, mhd.py:225-231).  The arithmetic
runs in the fused sm_100a stencil (``csrc/stencil.cu``) and is bitwise equal to
the reference's NumPy evaluation.

Container policy: a ``StateGrid`` may hold a NumPy array (reference-style,
host buffers: copied to the device per call) or a CUDA float64 tensor
(device-resident, no copies).  Results come back in the container type of the
input.
"""

import ctypes
import struct
import threading
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from paper_2108_13622_b200 import _lib
from paper_2108_13622_b200 import _ops
from paper_2108_13622_b200.linearize import RhsBlowupError

RHO, MX, MY, MZ, BX, BY, BZ, EN = range(8)
NVAR = 8
FIELD_NAMES = ("rho", "mx", "my", "mz", "bx", "by", "bz", "en")

_MAGIC = b"XMHD"
_FORMAT_VERSION = 1
_HEADER = "<4sIIIIddd"


class Boundary(Enum):
    PERIODIC = "periodic"
    REFLECTING = "reflecting"


@dataclass
class MHDParams:
    """Dimensionless coefficients: mu = 1/Re, eta = 1/S, kappa = 1/Pr (mhd.py:39-48)."""
    mu: float
    eta: float
    kappa: float
    gamma: float = 5.0 / 3.0
    mu0: float = 1.0
    bc_x: Boundary = Boundary.PERIODIC
    bc_y: Boundary = Boundary.PERIODIC


@dataclass
class StateGrid:
    """Conserved fields on a uniform grid; data has shape (8, ny, nx) (mhd.py:51-70)."""
    nx: int
    ny: int
    dx: float
    dy: float
    data: object

    @classmethod
    def zeros(cls, nx, ny, dx, dy, device=None):
        if device is None:
            return cls(nx=nx, ny=ny, dx=dx, dy=dy, data=np.zeros((NVAR, ny, nx)))
        return cls(nx=nx, ny=ny, dx=dx, dy=dy,
                   data=torch.zeros((NVAR, ny, nx), dtype=torch.float64, device=device))

    def flat(self):
        return self.data.reshape(-1)

    def with_flat(self, flat):
        """Same geometry, fields taken from a flat state vector (kept on its device)."""
        if torch.is_tensor(flat):
            data = flat.reshape(NVAR, self.ny, self.nx)
        else:
            data = np.asarray(flat, dtype=float).reshape(NVAR, self.ny, self.nx)
        return StateGrid(nx=self.nx, ny=self.ny, dx=self.dx, dy=self.dy, data=data)

    def to_device(self):
        return StateGrid(self.nx, self.ny, self.dx, self.dy,
                         _ops.as_device(self.data).reshape(NVAR, self.ny, self.nx))


def _bc_code(b):
    return _lib.BC_PERIODIC if b is Boundary.PERIODIC else _lib.BC_REFLECTING


_ctx_cache = {}
_ctx_lock = threading.Lock()


def context_for(nx, ny, dx, dy, params):
    """Native context for one geometry + parameter set (cached per device)."""
    _lib.require_cuda()
    key =(torch.cuda.current_device(), int(nx), int(ny), float(dx), float(dy),
           float(params.mu), float(params.eta), float(params.kappa), float(params.gamma),
           float(params.mu0), params.bc_x, params.bc_y)
    with _ctx_lock:
        c = _ctx_cache.get(key)
        if c is None:
            c = _lib.Context(nx, ny, dx, dy, params.mu, params.eta, params.kappa,
                             params.gamma, params.mu0, _bc_code(params.bc_x),
                             _bc_code(params.bc_y))
            _ctx_cache[key] = c
    return c


def _blowup_scan(f, nx, ny, j0=0):
    """(count, first <= 8 non-finite cells as (field, j + j0, i)) in C order."""
    host = _ops.to_host(f).reshape(NVAR, ny, nx)
    bad = np.argwhere(~np.isfinite(host))
    return len(bad), [(int(k), int(jj) + j0, int(ii)) for k, jj, ii in bad[:8]]


def _blowup_error(count, cells):
    """RhsBlowupError with the reference's message and cell list (mhd.py:225-231)
    from C-ordered (field, j, i) cells and the total count."""
    field, j, i = cells[0]
    return RhsBlowupError(
        f"non-finite rhs in field {FIELD_NAMES[field]} at cell "
        f"(i={i}, j={j}); {count} cells affected",
        cells=[(FIELD_NAMES[k], ii, jj) for k, jj, ii in cells[:8]])


def _blowup(f, nx, ny):
    """RhsBlowupError with the reference's message and cell list (mhd.py:225-231)."""
    return _blowup_error(*_blowup_scan(f, nx, ny))


def bad_cells_buffer():
    """int[XMHD_BAD_CELLS_LEN] out-parameter of xmhd_rhs / xmhd_jvp / xmhd_leja."""
    return (ctypes.c_int * _lib.BAD_CELLS_LEN)()


def decode_bad_cells(buf, j0=0):
    """(count, [(field, j + j0, i)]) from an XMHD_BAD_CELLS_LEN buffer."""
    cells = []
    for k in range(8):
        f, i, j = buf[1 + 3 * k], buf[2 + 3 * k], buf[3 + 3 * k]
        if f < 0:
            break
        cells.append((f, j + j0, i))
    return buf[0], cells


def blowup_from_cells(buf):
    """RhsBlowupError from the cells the C-ABI reported."""
    count, cells = decode_bad_cells(buf)
    if not cells:
        return RhsBlowupError("non-finite rhs (no cell reported)")
    return _blowup_error(count, cells)


class MhdRhs:
    """Device RHS bound to a geometry and MHDParams: flat u -> flat F(u).

    This is the B200 counterpart of the reference's
    ``lambda flat: mhd_rhs(geometry.with_flat(flat), params)`` (harness.py:129).
    Wrapped in an ``RhsOperator`` it also unlocks the fused JVP / Leja kernels.
    """

    def __init__(self, geometry, params):
        self.nx, self.ny = geometry.nx, geometry.ny
        self.dx, self.dy = geometry.dx, geometry.dy
        self.params = params
        self.n = NVAR * self.nx * self.ny
        self.ctx = context_for(self.nx, self.ny, self.dx, self.dy, params)

    def __call__(self, flat, out=None):
        u = _ops.as_device(flat).reshape(-1)
        if u.numel() != self.n:
            raise ValueError(f"state has {u.numel()} entries, grid needs {self.n}")
        if out is None:
            out = torch.empty_like(u)
        lib = _lib.load()
        bad = bad_cells_buffer()
        rc = lib.xmhd_rhs(self.ctx.bind_stream(), _lib.ptr(u), _lib.ptr(out), bad)
        _lib.check(rc, "xmhd_rhs")
        if rc == _lib.NONFINITE:
            raise blowup_from_cells(bad)
        return out


def mhd_rhs(state, params):
    """dU/dt of the resistive MHD equations as a flat vector (mhd.py:127-232)."""
    f = MhdRhs(state, params)(state.flat())
    return _ops.like(f, state.data)


def discrete_div_b(state, params):
    """Centred-difference divergence of (bx, by) at every cell (mhd.py:235-240)."""
    ctx = context_for(state.nx, state.ny, state.dx, state.dy, params)
    u = _ops.as_device(state.data).reshape(-1)
    field = torch.empty((state.ny, state.nx), dtype=torch.float64, device=u.device)
    _divb(ctx, u, field)
    return _ops.like(field, state.data)


def max_abs_div_b(state, params):
    """max |discrete_div_b| as a float (one device reduction)."""
    ctx = context_for(state.nx, state.ny, state.dx, state.dy, params)
    return _divb(ctx, _ops.as_device(state.data).reshape(-1), None)


def _divb(ctx, u, field):
    out = ctypes.c_double()
    rc = _lib.load().xmhd_divb(ctx.bind_stream(), _lib.ptr(u),
                               _lib.ptr(field) if field is not None else None,
                               ctypes.byref(out))
    _lib.check(rc, "xmhd_divb")
    return float(out.value)


def conserved_totals(state):
    """Cell-sum times cell-area of every conserved field (mhd.py:243-247)."""
    ctx = context_for(state.nx, state.ny, state.dx, state.dy, MHDParams(0.0, 0.0, 0.0))
    u = _ops.as_device(state.data).reshape(-1)
    out = (ctypes.c_double * 8)()
    _lib.check(_lib.load().xmhd_field_sums(ctx.bind_stream(), _lib.ptr(u), out),
               "xmhd_field_sums")
    area = state.dx * state.dy
    return {name: float(out[k]) * area for k, name in enumerate(FIELD_NAMES)}


def apply_bc(state, params):
    """Field data with one ghost layer per side filled from the boundaries (mhd.py:108-110)."""
    data = _ops.as_device(state.data).reshape(NVAR, state.ny, state.nx)
    padded = _pad_device(data, 1, params)
    return _ops.like(padded, state.data)


def _pad_device(data, g, params):
    """Ghost extension by index arithmetic (pure data movement + exact sign flips)."""
    nf, ny, nx = data.shape
    dev = data.device

    def index(n, bc):
        i = torch.arange(-g, n + g, device=dev)
        sign = torch.ones(n + 2 * g, dtype=torch.float64, device=dev)
        if bc is Boundary.PERIODIC:
            return torch.remainder(i, n), None
        lo = i < 0
        hi = i >= n
        src = torch.where(lo, -1 - i, torch.where(hi, 2 * n - 1 - i, i))
        sign[lo | hi] = -1.0
        return src, sign

    ix, sx = index(nx, params.bc_x)
    iy, sy = index(ny, params.bc_y)
    out = data[:, iy][:, :, ix].clone()
    if sx is not None:
        for f in (MX, BX):
            out[f] *= sx
    if sy is not None:
        for f in (MY, BY):
            out[f] *= sy[:, None]
    return out


def write_checkpoint(path, state, time):
    """Binary checkpoint: magic, version, nx, ny, nvar, time, dx, dy, planes (mhd.py:250-257)."""
    host = _ops.to_host(state.data) if torch.is_tensor(state.data) else np.asarray(state.data)
    header = struct.pack(_HEADER, _MAGIC, _FORMAT_VERSION, state.nx, state.ny, NVAR, time,
                         state.dx, state.dy)
    with open(path, "wb") as fh:
        fh.write(header)
        for k in range(NVAR):
            fh.write(np.ascontiguousarray(host[k], dtype="<f8").tobytes())


def read_checkpoint(path):
    """Read a checkpoint written by write_checkpoint; returns (StateGrid, time) (mhd.py:260-273)."""
    with open(path, "rb") as fh:
        header = fh.read(struct.calcsize(_HEADER))
        magic, version, nx, ny, nvar, time, dx, dy = struct.unpack(_HEADER, header)
        if magic != _MAGIC:
            raise ValueError(f"not a checkpoint file: bad magic {magic!r}")
        if version != _FORMAT_VERSION:
            raise ValueError(f"unsupported checkpoint version {version}")
        if nvar != NVAR:
            raise ValueError(f"expected {NVAR} fields, file has {nvar}")
        raw = np.frombuffer(fh.read(nvar * ny * nx * 8), dtype="<f8")
    return StateGrid(nx=nx, ny=ny, dx=dx, dy=dy, data=raw.reshape(nvar, ny, nx).astype(float)), time
