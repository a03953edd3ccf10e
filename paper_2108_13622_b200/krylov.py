"""Arnoldi/Krylov phi-actions on the B200 — the paper's comparison baseline.

Host mirror of the reference module ``pkg/src/xmhd/krylov.py`` (same names,
signature, result type and errors).  The basis vectors live in HBM (one
device vector per Arnoldi step, at most 201), each matvec is the fused FD-JVP
stencil, and both modified Gram-Schmidt passes of a step run as a chain of
stream-ordered device updates (``xmhd_krylov_mgs``: each launch subtracts the
previous projection and reduces the next dot product, 32 B per element), so
the host synchronises once per Arnoldi step.  The (m+1) x m Hessenberg matrix
and phi_l(dt H) e1 are small dense host work, as in the reference.
"""

import ctypes
import math

import numpy as np
import torch

from paper_2108_13622_b200 import _lib
from paper_2108_13622_b200 import _ops
from paper_2108_13622_b200.leja import PhiApplyResult
from paper_2108_13622_b200.phi import _check_order

M_DEFAULT = 100       # krylov.py:15
M_CAP = 200           # krylov.py:16
_TAYLOR_DEGREE = 30   # phi.py:19
_TAYLOR_RADIUS = 3.5  # phi.py:20


def _expm_taylor(a):
    """exp(a) of a small dense matrix by scaling and squaring (phi.py:50-60)."""
    norm = np.linalg.norm(a, 1)
    s = int(math.ceil(math.log2(max(1.0, norm / _TAYLOR_RADIUS))))
    b = a / (2.0 ** s)
    f = np.eye(a.shape[0])
    for k in range(_TAYLOR_DEGREE, 0, -1):
        f = np.eye(a.shape[0]) + (b @ f) / k
    for _ in range(s):
        f = f @ f
    return f


def _phi_e1(l, h):
    """phi_l(H) e1 for a small dense H via an augmented exponential (krylov.py:19-31)."""
    m = h.shape[0]
    if l == 0:
        return _expm_taylor(h)[:, 0]
    dim = m + l
    aug = np.zeros((dim, dim))
    aug[:m, :m] = h
    aug[0, m] = 1.0
    for k in range(l - 1):
        aug[m + k, m + k + 1] = 1.0
    return _expm_taylor(aug)[:m, dim - 1]


def _ptrs(vecs):
    return (ctypes.c_void_p * len(vecs))(*[ctypes.c_void_p(v.data_ptr()) for v in vecs])


def _mgs_local(h, basis, w, coef):
    """Both MGS passes on one device; returns sum(w^2) afterwards."""
    nb = len(basis)
    out = (ctypes.c_double * (2 * nb))()
    ssq = ctypes.c_double()
    rc = _lib.load().xmhd_krylov_mgs(h, _ptrs(basis), nb, _lib.ptr(w), w.numel(), out,
                                     ctypes.byref(ssq))
    _lib.check(rc, "xmhd_krylov_mgs")
    coef[:] = np.frombuffer(out, dtype=np.float64).reshape(2, nb)
    return float(ssq.value)


def _mgs_reduced(h, basis, w, coef, red):
    """Both MGS passes on a y-strip: every coefficient is reduced over the ranks."""
    lib = _lib.load()
    n = w.numel()
    part = ctypes.c_double()

    def update(v, c, nxt):
        rc = lib.xmhd_mgs_update(h, _lib.ptr(w), n, _lib.ptr(v) if v is not None else None,
                                 float(c), _lib.ptr(nxt) if nxt is not None else None,
                                 ctypes.byref(part))
        _lib.check(rc, "xmhd_mgs_update")
        return red.sum([part.value])[0]

    nb = len(basis)
    c = update(None, 0.0, basis[0])
    for p in range(2):
        for i in range(nb):
            coef[p, i] = c
            nxt = basis[i + 1] if i + 1 < nb else (basis[0] if p == 0 else None)
            c = update(basis[i], coef[p, i], nxt)
    return c


def apply_phi_krylov(l, matvec, v, dt, tol, m_max=M_DEFAULT):
    """Approximate phi_l(J dt) v by Arnoldi projection (krylov.py:34-84).

    The basis grows from v/||v||; after each expansion phi_l(dt H_m) is
    evaluated on the projected Hessenberg matrix and the residual surrogate
    ||v|| * |h_{m+1,m}| * |(phi_l(dt H_m))_{m,1}| * dt decides convergence.
    Happy breakdown counts as exact convergence.
    """
    _check_order(l)
    if tol <= 0:
        raise ValueError("tolerance must be positive")
    if m_max > M_CAP:
        raise ValueError(f"m_max exceeds the cap of {M_CAP}")
    host_io = _ops.is_host(v)
    vd = _ops.as_device(v).reshape(-1)
    beta = _ops.norm(vd)
    if beta == 0:
        raise ValueError("cannot build a Krylov space from the zero vector")
    red = _ops.reducer()
    n = int(_ops.global_sum([float(vd.numel())])[0])
    m_max = min(m_max, n)
    ctx = _ops.util_ctx()
    h = ctx.bind_stream()

    hess = np.zeros((m_max + 1, m_max))
    basis = [_ops.divide(vd, beta)]
    coef = np.zeros((2, m_max + 1))
    matvecs = 0
    phicol = None
    residual = np.inf
    for j in range(m_max):
        y = basis[j]
        w = matvec(_ops.to_host(y) if host_io else y)
        matvecs += 1
        wd = _ops.as_device(w).reshape(-1)
        if any(wd.data_ptr() == b.data_ptr() for b in basis) or wd.data_ptr() == vd.data_ptr():
            wd = wd.clone()   # w is updated in place below
        nb = j + 1
        c = coef[:, :nb]
        ssq = _mgs_local(h, basis, wd, c) if red is None else _mgs_reduced(h, basis, wd, c, red)
        for i in range(nb):        # hess[i, j] += c, pass by pass (krylov.py:63,67)
            hess[i, j] += c[0, i]
        for i in range(nb):
            hess[i, j] += c[1, i]
        hnext = math.sqrt(ssq)
        hess[j + 1, j] = hnext
        m = j + 1
        phicol = _phi_e1(l, dt * hess[:m, :m])
        residual = beta * hnext * abs(phicol[m - 1]) * dt
        breakdown = hnext <= 1e-14 * max(1.0, np.abs(hess[:m, :m]).max())
        if breakdown or residual <= tol or m == n:
            out = _combine(h, basis[:m], phicol, beta)
            return PhiApplyResult(vector=_ops.like(out, v), iterations=matvecs, converged=True,
                                  residual=0.0 if breakdown else residual)
        basis.append(_ops.divide(wd, hnext, out=wd))
    out = _combine(h, basis[:m_max], phicol, beta)
    return PhiApplyResult(vector=_ops.like(out, v), iterations=matvecs, converged=False,
                          residual=residual)


def _combine(h, basis, phicol, beta):
    """beta * (V_m^T phicol) on the device (krylov.py:79-80)."""
    out = torch.empty_like(basis[0])
    cs = np.ascontiguousarray(phicol, dtype=np.float64)
    rc = _lib.load().xmhd_krylov_combine(h, _ptrs(basis),
                                         cs.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                         len(basis), float(beta), out.numel(), _lib.ptr(out))
    _lib.check(rc, "xmhd_krylov_combine")
    return out
