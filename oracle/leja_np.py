"""NumPy restatement of the reference's Leja / divided-difference / JVP machinery.

Test infrastructure only (see ``oracle/__init__.py``).  Follows:

* Leja points on [-2, 2] ......................... leja.py:24-53
* shift / scale .................................. leja.py:63-72
* phi_l divided differences (bidiagonal route) ... phi.py:99-144
* Newton coefficient cache (l, q, theta) ......... leja.py:84-100
* Newton/Leja recurrence ......................... leja.py:103-150
* FD Jacobian action ............................. linearize.py:15, 56-67
* power-iteration spectral estimate .............. linearize.py:88-135
"""

import math
from dataclasses import dataclass, field

import numpy as np

N_LEJA = 500          # leja.py:15
GRID_PTS = 10001      # leja.py:18
SQRT_EPS = math.sqrt(np.finfo(float).eps)   # linearize.py:15
POWER_TOL = 0.02      # linearize.py:22
POWER_MAXIT = 100     # linearize.py:23

_points = None


def leja_points(count=N_LEJA):
    """Sequential argmax of the log-distance product over a uniform grid."""
    global _points
    if not 1 <= count <= N_LEJA:
        raise ValueError(count)
    if _points is None:
        cand = np.linspace(-2.0, 2.0, GRID_PTS)
        out = np.empty(N_LEJA)
        out[0] = 2.0
        with np.errstate(divide="ignore"):
            acc = np.log(np.abs(cand - out[0]))
            for k in range(1, N_LEJA):
                top = acc.max()
                near = np.nonzero(acc >= top - 1e-12 * max(1.0, abs(top)))[0]
                out[k] = cand[near[np.argmax(cand[near])]]
                acc += np.log(np.abs(cand - out[k]))
        _points = out
    return _points[:count]


def shift_scale(alpha):
    """(q, theta) placing [-alpha, 0] onto [-2, 2] (leja.py:63-72)."""
    if alpha <= 0:
        raise ValueError(alpha)
    return -0.5 * alpha, 0.25 * alpha


def phi_divdiff(l, nodes, subdiag=1.0):
    """First column of phi_l of the lower-bidiagonal node matrix (phi.py:99-144)."""
    nodes = np.asarray(nodes, dtype=float)
    diag_full = np.concatenate([np.zeros(l), nodes])
    n = diag_full.size
    nterm = 60
    big = max(np.max(np.abs(diag_full)), abs(subdiag), 1e-30)
    s = max(0, int(math.ceil(math.log2(big))),
            int(math.ceil(math.log2((n + nterm) / nterm))))
    d = diag_full / 2.0 ** s
    e = subdiag / 2.0 ** s

    def bidiag_apply(w):
        r = d * w
        r[1:] += e * w[:-1]
        return r

    col = np.zeros(n)
    col[0] = 1.0
    for _ in range(2 ** s):
        t = col.copy()
        acc = col.copy()
        for k in range(1, nterm):
            t = bidiag_apply(t) / k
            acc += t
        col = acc
    return col[l:]


class CoeffCache:
    """Per-(l, q, theta) coefficient cache with the reference's FIFO policy."""

    def __init__(self):
        self.store = {}

    def get(self, l, q, theta, count):
        key = (l, q, theta)
        hit = self.store.get(key)
        if hit is not None and hit.size >= count:
            return hit
        xi = leja_points(N_LEJA)[:count]
        c = phi_divdiff(l, q + theta * xi, subdiag=theta) / theta ** l
        if len(self.store) > 64:
            self.store.pop(next(iter(self.store)))
        self.store[key] = c
        return c


GLOBAL_CACHE = CoeffCache()


@dataclass
class LejaOut:
    vector: np.ndarray
    iterations: int
    converged: bool
    residual: float


def phi_leja(l, matvec, v, dt, q, theta, tol, cache=None):
    """phi_l(J dt) v by Newton interpolation at Leja points (leja.py:103-150)."""
    cache = GLOBAL_CACHE if cache is None else cache
    if tol <= 0:
        raise ValueError(tol)
    xi = leja_points(N_LEJA)
    n_c = 64
    c = cache.get(l, q, theta, n_c)
    y = np.array(v, dtype=float, copy=True)
    limit = 1e120 * max(1.0, np.linalg.norm(y))
    p = c[0] * y
    count = 0
    resid = np.inf
    prev_small = False
    for m in range(1, N_LEJA):
        if m >= c.size:
            n_c = min(2 * n_c, N_LEJA)
            c = cache.get(l, q, theta, n_c)
        w = matvec(y)
        count += 1
        y = (dt * w - q * y) / theta - xi[m - 1] * y
        ny = np.linalg.norm(y)
        if not np.isfinite(ny) or ny > limit:
            return LejaOut(p, count, False, np.inf)
        p = p + c[m] * y
        resid = abs(c[m]) * ny / max(1.0, np.linalg.norm(p))
        if resid <= tol:
            if prev_small:
                return LejaOut(p, count, True, resid)
            prev_small = True
        else:
            prev_small = False
    return LejaOut(p, count, False, resid)


class CountedRhs:
    """Mirror of RhsOperator (linearize.py:34-43)."""

    def __init__(self, fn):
        self.fn = fn
        self.calls = 0

    def __call__(self, u):
        self.calls += 1
        return self.fn(u)


class Frozen:
    """Mirror of FrozenLinearization (linearize.py:46-53)."""

    def __init__(self, rhs, u):
        self.rhs = rhs
        self.u = np.asarray(u, dtype=float)
        self.fu = np.asarray(rhs(self.u), dtype=float)
        self.unorm = np.linalg.norm(self.u)


def fd_jvp(lin, w):
    """Forward-difference Jacobian action (linearize.py:56-67)."""
    w = np.asarray(w, dtype=float)
    wn = np.linalg.norm(w)
    if wn == 0.0:
        return np.zeros_like(lin.u)
    eps = SQRT_EPS * max(1.0, lin.unorm) / max(wn, 1e-300)
    return (lin.rhs(lin.u + eps * w) - lin.fu) / eps


@dataclass
class Spectrum:
    alpha: float
    age_steps: int = 0
    interval: int = 50
    safety: float = 1.25
    vector: np.ndarray | None = field(default=None, repr=False)
    mags: list = field(default_factory=list, repr=False)


def power_alpha(lin, prev=None, interval=50, safety=1.25, rng=None):
    """Cached, warm-started power iteration (linearize.py:88-135)."""
    if prev is not None:
        interval, safety = prev.interval, prev.safety
        if prev.age_steps + 1 < prev.interval:
            return Spectrum(prev.alpha, prev.age_steps + 1, interval, safety,
                            prev.vector, prev.mags)
    n = lin.u.size
    if prev is not None and prev.vector is not None and prev.vector.size == n:
        w = prev.vector
    else:
        rng = np.random.default_rng(0) if rng is None else rng
        w = rng.standard_normal(n)
    wn = np.linalg.norm(w)
    if wn == 0.0:
        w = np.ones(n)
        wn = np.linalg.norm(w)
    w = w / wn
    mags = []
    for _ in range(POWER_MAXIT):
        jw = fd_jvp(lin, w)
        mag = np.linalg.norm(jw)
        if mag < 1e-300 or not np.isfinite(mag):
            return Spectrum(0.0, 0, interval, safety, None, mags)
        mags.append(mag)
        w = jw / mag
        if len(mags) >= 3 and (abs(mag - mags[-2]) <= POWER_TOL * mag
                               or abs(mag - mags[-3]) <= POWER_TOL * mag):
            break
    return Spectrum(safety * max(mags[-3:]), 0, interval, safety, w, mags)
