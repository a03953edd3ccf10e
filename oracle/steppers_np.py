"""NumPy restatement of the reference's exponential Rosenbrock steppers,
step-size controllers and adaptive driver loop.

Test infrastructure only (see ``oracle/__init__.py``).  Follows:

* error_norm ........................ integrators.py:88-96
* _PhiBroker ........................ integrators.py:99-136
* _stage_difference ................. integrators.py:146-153
* EXP/ROS-Euler, EXPRB43, EXPRB54s4 . integrators.py:139-143, 156-199
* step .............................. integrators.py:284-320
* controllers ....................... controllers.py:14-80
* adaptive run loop ................. harness.py:105-249
"""

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

from oracle import krylov_np as kr
from oracle import leja_np as lj
from oracle import mhd_np

ORDERS = {"exp-euler": (1, None), "ros-euler": (2, None),
          "exprb43": (4, 3), "exprb54s4": (5, 4)}

# controllers.py:14-23
ALPHA_C = 0.65241444
BETA_C = 0.26862269
LAMBDA_C = 1.37412002
DELTA_C = 0.64446017
SAFETY = 0.9
GROWTH = 2.0


def rel_err(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    if a.shape != b.shape:
        raise ValueError("shape")
    top = np.linalg.norm(a - b)
    bot = np.linalg.norm(b)
    return top if bot == 0.0 else top / bot


class Broker:
    def __init__(self, lin, dt, alpha, tol, cache=None, method="leja"):
        self.lin, self.dt, self.alpha, self.tol = lin, dt, alpha, tol
        self.method = method
        self.apps = 0
        self.iters = 0
        self.failed = False
        self.cache = cache

    def apply(self, l, c, vec):
        self.apps += 1
        if self.alpha < 1e-14:
            return vec / math.factorial(l)
        h = c * self.dt
        if self.method == "krylov":            # integrators.py:129-130
            r = kr.phi_krylov(l, lambda w: lj.fd_jvp(self.lin, w), vec, h, self.tol)
        else:
            q, th = lj.shift_scale(self.alpha * h)
            r = lj.phi_leja(l, lambda w: lj.fd_jvp(self.lin, w), vec, h, q, th,
                            self.tol, self.cache)
        self.iters += r.iterations
        if not r.converged:
            self.failed = True
        return r.vector


def stage_diff(lin, rhs, s, u, fu):
    return (np.asarray(rhs(s), dtype=float) - fu) - lj.fd_jvp(lin, s - u)


def _euler(lin, br, u, dt, rhs):
    return u + dt * br.apply(1, 1.0, lin.fu), 0.0


def _exprb43(lin, br, u, dt, rhs):
    fu = lin.fu
    a = u + 0.5 * dt * br.apply(1, 0.5, fu)
    da = stage_diff(lin, rhs, a, u, fu)
    p1 = br.apply(1, 1.0, fu)
    b = u + dt * p1 + dt * br.apply(1, 1.0, da)
    db = stage_diff(lin, rhs, b, u, fu)
    w3 = 16.0 * da - 2.0 * db
    w4 = -48.0 * da + 12.0 * db
    u3 = u + dt * p1 + dt * br.apply(3, 1.0, w3)
    u4 = u3 + dt * br.apply(4, 1.0, w4)
    return u4, rel_err(u3, u4)


def _exprb54s4(lin, br, u, dt, rhs):
    fu = lin.fu
    a = u + 0.25 * dt * br.apply(1, 0.25, fu)
    da = stage_diff(lin, rhs, a, u, fu)
    b = (u + 0.5 * dt * br.apply(1, 0.5, fu)
         + 4.0 * dt * br.apply(3, 0.5, da))
    db = stage_diff(lin, rhs, b, u, fu)
    c = (u + 0.9 * dt * br.apply(1, 0.9, fu)
         + (729.0 / 125.0) * dt * br.apply(3, 0.9, db))
    dc = stage_diff(lin, rhs, c, u, fu)
    w1 = 64.0 * da - 8.0 * db
    w2 = -60.0 * da - (285.0 / 8.0) * db + (125.0 / 8.0) * dc
    w3 = 18.0 * db - (250.0 / 81.0) * dc
    w4 = -60.0 * db + (500.0 / 27.0) * dc
    p1 = br.apply(1, 1.0, fu)
    u4 = (u + dt * p1 + dt * br.apply(3, 1.0, w1)
          + dt * br.apply(4, 1.0, w2))
    u5 = (u + dt * p1 + dt * br.apply(3, 1.0, w3)
          + dt * br.apply(4, 1.0, w4))
    return u5, rel_err(u4, u5)


def _epirk5p1(lin, br, u, dt, rhs):
    """integrators.py:56-75, 202-222."""
    a11, a21, a22 = 0.35129592695058193092, 0.84405472011657126298, 1.6905891609568963624
    b1, b2, b3 = 1.0, 1.2727127317356892397, 2.271459926542262275
    g11, g21, g22, g31 = a11, a21, 0.5, 1.0
    g32, g33, g32e, g33e = 0.71111095364366870359, 0.62378111953371494809, 0.5, 1.0
    fu = lin.fu
    a = u + a11 * dt * br.apply(1, g11, fu)
    da = stage_diff(lin, rhs, a, u, fu)
    b = (u + a21 * dt * br.apply(1, g21, fu) + a22 * dt * br.apply(1, g22, da))
    db = stage_diff(lin, rhs, b, u, fu)
    w = db - 2.0 * da
    p1 = br.apply(1, g31, fu)
    u5 = (u + b1 * dt * p1 + b2 * dt * br.apply(1, g32, da) + b3 * dt * br.apply(3, g33, w))
    u4 = (u + b1 * dt * p1 + b2 * dt * br.apply(1, g32e, da) + b3 * dt * br.apply(3, g33e, w))
    return u5, rel_err(u4, u5)


SCHEMES = {"exp-euler": _euler, "ros-euler": _euler,
           "exprb43": _exprb43, "exprb54s4": _exprb54s4, "epirk5p1": _epirk5p1}

# explicit embedded pairs, integrators.py:225-281 (Zonneveld 4(3), Dormand-Prince 5(4))
_TAB = {
    "rk43": ([[], [0.5], [0.0, 0.5], [0.0, 0.0, 1.0],
              [5.0 / 32.0, 7.0 / 32.0, 13.0 / 32.0, -1.0 / 32.0]],
             [1.0 / 6.0, 1.0 / 3.0, 1.0 / 3.0, 1.0 / 6.0, 0.0],
             [-0.5, 7.0 / 3.0, 7.0 / 3.0, 13.0 / 6.0, -16.0 / 3.0]),
    "dopri54": ([[], [0.2], [3.0 / 40.0, 9.0 / 40.0], [44.0 / 45.0, -56.0 / 15.0, 32.0 / 9.0],
                 [19372.0 / 6561.0, -25360.0 / 2187.0, 64448.0 / 6561.0, -212.0 / 729.0],
                 [9017.0 / 3168.0, -355.0 / 33.0, 46732.0 / 5247.0, 49.0 / 176.0,
                  -5103.0 / 18656.0],
                 [35.0 / 384.0, 0.0, 500.0 / 1113.0, 125.0 / 192.0, -2187.0 / 6784.0,
                  11.0 / 84.0]],
                [35.0 / 384.0, 0.0, 500.0 / 1113.0, 125.0 / 192.0, -2187.0 / 6784.0,
                 11.0 / 84.0, 0.0],
                [5179.0 / 57600.0, 0.0, 7571.0 / 16695.0, 393.0 / 640.0, -92097.0 / 339200.0,
                 187.0 / 2100.0, 1.0 / 40.0]),
}
ORDERS.update({"epirk5p1": (5, 4), "rk43": (4, 3), "dopri54": (5, 4)})


def _explicit(scheme, rhs, u, dt):
    a, b, bhat = _TAB[scheme]
    ks = []
    for row in a:
        x = u
        for cf, kj in zip(row, ks):
            if cf != 0.0:
                x = x + dt * cf * kj
        ks.append(np.asarray(rhs(x), dtype=float))
    hi = u + dt * sum(bi * ki for bi, ki in zip(b, ks) if bi != 0.0)
    lo = u + dt * sum(bi * ki for bi, ki in zip(bhat, ks) if bi != 0.0)
    return hi, rel_err(lo, hi)


@dataclass
class StepOut:
    new_state: np.ndarray
    error_estimate: float
    rhs_calls: int
    phi_iterations: int
    phi_applications: int
    converged: bool


def one_step(scheme, rhs, u, dt, alpha, tol, lin=None, cache=None, method="leja"):
    if dt <= 0:
        raise ValueError("dt")
    u = np.asarray(u, dtype=float)
    before = rhs.calls
    if scheme in _TAB:
        try:
            un, err = _explicit(scheme, rhs, u, dt)
            ok = np.all(np.isfinite(un)) and np.isfinite(err)
        except (mhd_np.NonFiniteRhs, FloatingPointError):
            un, err, ok = u, np.inf, False
        return StepOut(un, err, rhs.calls - before, 0, 0, bool(ok))
    mag = alpha.alpha if isinstance(alpha, lj.Spectrum) else float(alpha)
    if lin is None:
        lin = lj.Frozen(rhs, u)
    br = Broker(lin, dt, mag, tol, cache, method)
    try:
        un, err = SCHEMES[scheme](lin, br, u, dt, rhs)
        ok = (not br.failed) and np.all(np.isfinite(un)) and np.isfinite(err)
    except (mhd_np.NonFiniteRhs, FloatingPointError):
        un, err, ok = u, np.inf, False
    return StepOut(un, err, rhs.calls - before, br.iters, br.apps, bool(ok))


def trad_next(dt, err, tol, p):
    raw = SAFETY * dt * (tol / max(err, 1e-300)) ** (1.0 / (p + 1))
    return min(max(raw, dt / GROWTH), dt * GROWTH)


def cost_next(dt, dt_prev, cost, cost_prev):
    dl = math.log(dt) - math.log(dt_prev)
    if abs(dl) < 1e-12:
        return dt * LAMBDA_C
    slope = (math.log(cost) - math.log(cost_prev)) / dl
    s = math.exp(-ALPHA_C * math.tanh(BETA_C * slope))
    if 1.0 <= s < LAMBDA_C:
        return dt * LAMBDA_C
    if DELTA_C <= s < 1.0:
        return dt * DELTA_C
    return dt * s


@dataclass
class Rec:
    t: float
    dt: float
    error: float
    rhs_calls: int
    phi_iterations: int
    phi_applications: int
    accepted: bool
    cost: float


@dataclass
class Report:
    steps: list = field(default_factory=list)
    accepted: int = 0
    rejected: int = 0
    rhs_evals: int = 0
    phi_iterations: int = 0
    spectrum_rhs_evals: int = 0
    t_reached: float = 0.0
    status: str = "ok"
    final: np.ndarray | None = None
    checksum: str = ""
    max_divb: float = 0.0
    mass_drift: float = 0.0


def run(data0, dx, dy, mu, eta, kappa, scheme, tol, t_final, gamma=5.0 / 3.0,
        mu0=1.0, periodic_x=True, periodic_y=True, interval=50, seed=0,
        controller="combined", max_accepted=None, cache=None, method="leja"):
    """Adaptive driver loop of harness.py:123-249 on an explicit initial state.

    ``max_accepted`` stops cleanly after that many accepted steps (the
    BASELINE "N adaptive steps" configs); None reproduces the reference loop.
    """
    shape = data0.shape

    def f(flat):
        return mhd_np.rhs(flat.reshape(shape), dx, dy, mu, eta, kappa, gamma,
                          mu0, periodic_x, periodic_y)

    op = lj.CountedRhs(f)
    rng = np.random.default_rng(seed)
    p_ctrl = ORDERS[scheme][1] or ORDERS[scheme][0]
    u = data0.reshape(-1).copy()
    rep = Report()
    m0 = float(np.sum(data0[0])) * (dx * dy)
    rep.max_divb = float(np.max(np.abs(mhd_np.div_b(data0, dx, dy, periodic_x,
                                                      periodic_y))))
    t = 0.0
    dt = min(mhd_np.initial_dt(data0, dx, dy, gamma, mu0), t_final) if t_final > 0 else 0.0
    est = None
    dt_prev = cost_prev = None
    streak = 0
    while t < t_final - 1e-14 * max(1.0, t_final):
        if max_accepted is not None and rep.accepted >= max_accepted:
            break
        dt = min(dt, t_final - t)
        c0 = op.calls
        lin = lj.Frozen(op, u)
        cs = op.calls
        est = lj.power_alpha(lin, est, interval=interval, rng=rng)
        rep.spectrum_rhs_evals += op.calls - cs
        while True:
            cb = op.calls
            res = one_step(scheme, op, u, dt, est, tol, lin, cache, method)
            spent = op.calls - cb
            if res.converged and res.error_estimate <= tol:
                break
            rep.rejected += 1
            streak += 1
            rep.steps.append(Rec(t, dt, res.error_estimate, spent, res.phi_iterations,
                                 res.phi_applications, False, spent / dt))
            if streak >= 10:
                rep.status = "failed: too many consecutive rejections"
                break
            if not res.converged:
                dt = 0.5 * dt
            else:
                dt = trad_next(dt, res.error_estimate, tol, p_ctrl)
        if rep.status != "ok":
            break
        streak = 0
        t = t + dt
        u = res.new_state
        err = res.error_estimate
        i_n = op.calls - c0
        cost = i_n / dt
        rep.accepted += 1
        rep.phi_iterations += res.phi_iterations
        rep.steps.append(Rec(t, dt, err, i_n, res.phi_iterations,
                             res.phi_applications, True, cost))
        dvb = float(np.max(np.abs(mhd_np.div_b(u.reshape(shape), dx, dy,
                                                periodic_x, periodic_y))))
        rep.max_divb = max(rep.max_divb, dvb)
        dtt = trad_next(dt, err, tol, p_ctrl)
        if controller == "traditional" or dt_prev is None:
            dtn = dtt
        else:
            dtc = cost_next(dt, dt_prev, cost, cost_prev)
            dtn = dtc if controller == "cost" else min(dtc, dtt)
        dt_prev, cost_prev = dt, cost
        dt = dtn
        if not np.all(np.isfinite(u)):
            rep.status = "failed: non-finite state"
            break
    rep.t_reached = t
    rep.rhs_evals = op.calls
    rep.final = u.reshape(shape)
    rep.checksum = hashlib.sha256(np.ascontiguousarray(u, dtype="<f8").tobytes()).hexdigest()
    m1 = float(np.sum(rep.final[0])) * (dx * dy)
    rep.mass_drift = abs(m1 - m0) / abs(m0) if m0 else 0.0
    return rep
