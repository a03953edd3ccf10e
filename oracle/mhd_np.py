"""NumPy restatement of the reference's resistive-MHD right-hand side.

Test infrastructure only (see ``oracle/__init__.py``).  Follows
``pkg/src/xmhd/mhd.py`` of the reference:

* field order and (8, ny, nx) layout ............ mhd.py:26-28, 51-70
* ghost extension (periodic / mirror) ........... mhd.py:77-105
* centred differences, host-folded 2*dx ......... mhd.py:113-124
* ideal + diffusive fluxes, op order ............ mhd.py:127-223
* non-finite detection .......................... mhd.py:225-231
* div B, totals, checkpoint format .............. mhd.py:235-273

Every arithmetic step is one NumPy ufunc so the IEEE operation sequence equals
the reference's; the result is bitwise identical to ``xmhd.mhd.mhd_rhs``.
"""

import struct

import numpy as np

NFIELD = 8
I_RHO, I_MX, I_MY, I_MZ, I_BX, I_BY, I_BZ, I_EN = range(NFIELD)
NAMES = ("rho", "mx", "my", "mz", "bx", "by", "bz", "en")


class NonFiniteRhs(ArithmeticError):
    """Mirror of ``xmhd.linearize.RhsBlowupError`` (linearize.py:26-31)."""

    def __init__(self, message, cells=None):
        super().__init__(message)
        self.cells = cells


def _odd_fields(axis):
    # mhd.py:77-85: wall-normal momentum and field flip sign at a mirror wall
    return (I_MX, I_BX) if axis == "x" else (I_MY, I_BY)


def _mirror_sign(axis):
    s = np.ones((NFIELD, 1, 1))
    for f in _odd_fields(axis):
        s[f] = -1.0
    return s


def extend(q, g, periodic_x=True, periodic_y=True):
    """(8, ny, nx) -> (8, ny+2g, nx+2g) ghost-extended copy (mhd.py:88-105)."""
    if periodic_x:
        q = np.concatenate([q[:, :, q.shape[2] - g:], q, q[:, :, :g]], axis=2)
    else:
        s = _mirror_sign("x")
        lo = q[:, :, :g][:, :, ::-1]
        hi = q[:, :, q.shape[2] - g:][:, :, ::-1]
        q = np.concatenate([s * lo, q, s * hi], axis=2)
    if periodic_y:
        q = np.concatenate([q[:, q.shape[1] - g:, :], q, q[:, :g, :]], axis=1)
    else:
        s = _mirror_sign("y")
        lo = q[:, :g, :][:, ::-1, :]
        hi = q[:, q.shape[1] - g:, :][:, ::-1, :]
        q = np.concatenate([s * lo, q, s * hi], axis=1)
    return q


def cdx(a, two_dx):
    """x-centred difference on the interior of the last two axes (mhd.py:113-115)."""
    return (a[..., 1:-1, 2:] - a[..., 1:-1, :-2]) / two_dx


def cdy(a, two_dy):
    """y-centred difference on the interior of the last two axes (mhd.py:118-120)."""
    return (a[..., 2:, 1:-1] - a[..., :-2, 1:-1]) / two_dy


def inner(a):
    return a[..., 1:-1, 1:-1]


def rhs(data, dx, dy, mu, eta, kappa, gamma=5.0 / 3.0, mu0=1.0,
        periodic_x=True, periodic_y=True, check=True):
    """dU/dt of the resistive MHD system, shape (8, ny, nx) (mhd.py:127-232).

    Returned as a flat vector like the reference.  Raises NonFiniteRhs with the
    first <= 8 bad cells in C order when ``check`` is set (mhd.py:225-231).
    """
    data = np.asarray(data, dtype=float)
    nf, ny, nx = data.shape
    assert nf == NFIELD
    h2x = 2.0 * dx
    h2y = 2.0 * dy
    gm1 = gamma - 1.0
    with np.errstate(all="ignore"):
        q = extend(data, 2, periodic_x, periodic_y)
        rho, en = q[I_RHO], q[I_EN]
        bx, by, bz = q[I_BX], q[I_BY], q[I_BZ]
        v = q[I_MX:I_MZ + 1] / rho
        vx, vy, vz = v[0], v[1], v[2]
        bsq = bx * bx + by * by + bz * bz
        ekin = 0.5 * rho * (vx * vx + vy * vy + vz * vz)
        pgas = gm1 * (en - ekin - 0.5 * bsq / mu0)
        pstar = pgas + 0.5 * bsq / mu0
        bv = bx * vx + by * vy + bz * vz
        ez = vy * bx - by * vx

        # ideal flux cubes on the 2-ghost grid, mhd.py:159-176
        fx = np.zeros_like(q)
        fy = np.zeros_like(q)
        fx[I_RHO] = rho * vx
        fy[I_RHO] = rho * vy
        fx[I_MX] = rho * vx * vx + pstar - bx * bx / mu0
        fy[I_MX] = rho * vy * vx - by * bx / mu0
        fx[I_MY] = rho * vx * vy - bx * by / mu0
        fy[I_MY] = rho * vy * vy + pstar - by * by / mu0
        fx[I_MZ] = rho * vx * vz - bx * bz / mu0
        fy[I_MZ] = rho * vy * vz - by * bz / mu0
        fy[I_BX] = ez
        fx[I_BY] = -ez
        fx[I_BZ] = vx * bz - bx * vz
        fy[I_BZ] = vy * bz - by * vz
        fx[I_EN] = (en + pstar) * vx - bx * bv / mu0
        fy[I_EN] = (en + pstar) * vy - by * bv / mu0
        res = -cdx(inner(fx), h2x)
        res -= cdy(inner(fy), h2y)

        # diffusive fluxes on the level-1 ring, mhd.py:181-223
        if mu != 0.0 or eta != 0.0 or kappa != 0.0:
            gvx = cdx(v, h2x)
            gvy = cdy(v, h2y)
            dv = gvx[0] + gvy[1]
            sxx = 2.0 * gvx[0] - (2.0 / 3.0) * dv
            syy = 2.0 * gvy[1] - (2.0 / 3.0) * dv
            sxy = gvy[0] + gvx[1]
            sxz = gvx[2]
            syz = gvy[2]
            jz = eta * (cdx(by, h2x) - cdy(bx, h2y))
            bzx = cdx(bz, h2x)
            bzy = cdy(bz, h2y)
            ux1, uy1, uz1 = inner(vx), inner(vy), inner(vz)
            kcond = mu * kappa * gamma / (gamma - 1.0)
            tmp = pgas / rho
            bx1, by1 = inner(bx), inner(by)
            bxx, bxy = cdx(bx, h2x), cdy(bx, h2y)
            byx, byy = cdx(by, h2x), cdy(by, h2y)
            gx = np.zeros((NFIELD,) + sxx.shape)
            gy = np.zeros((NFIELD,) + sxx.shape)
            gx[I_MX] = mu * sxx
            gy[I_MX] = mu * sxy
            gx[I_MY] = mu * sxy
            gy[I_MY] = mu * syy
            gx[I_MZ] = mu * sxz
            gy[I_MZ] = mu * syz
            gy[I_BX] = -jz
            gx[I_BY] = jz
            gx[I_BZ] = eta * bzx
            gy[I_BZ] = eta * bzy
            gx[I_EN] = (mu * (sxx * ux1 + sxy * uy1 + sxz * uz1)
                        + kcond * cdx(tmp, h2x)
                        + eta * (0.5 * cdx(bsq, h2x) - (bx1 * bxx + by1 * bxy)))
            gy[I_EN] = (mu * (sxy * ux1 + syy * uy1 + syz * uz1)
                        + kcond * cdy(tmp, h2y)
                        + eta * (0.5 * cdy(bsq, h2y) - (bx1 * byx + by1 * byy)))
            res += cdx(gx, h2x)
            res += cdy(gy, h2y)

    if check:
        bad_mask = ~np.isfinite(res)
        if bad_mask.any():
            bad = np.argwhere(bad_mask)
            f0, j0, i0 = bad[0]
            raise NonFiniteRhs(
                f"non-finite rhs in field {NAMES[f0]} at cell (i={i0}, j={j0}); "
                f"{len(bad)} cells affected",
                cells=[(NAMES[f], int(i), int(j)) for f, j, i in bad[:8]])
    return res.reshape(-1)


def div_b(data, dx, dy, periodic_x=True, periodic_y=True):
    """Centred div B at every interior cell (mhd.py:235-240)."""
    q = extend(np.asarray(data, dtype=float), 1, periodic_x, periodic_y)
    bx, by = q[I_BX], q[I_BY]
    return ((bx[1:-1, 2:] - bx[1:-1, :-2]) / (2.0 * dx)
            + (by[2:, 1:-1] - by[:-2, 1:-1]) / (2.0 * dy))


def totals(data, dx, dy):
    """Cell sums times cell area (mhd.py:243-247)."""
    area = dx * dy
    return {NAMES[k]: float(np.sum(data[k])) * area for k in range(NFIELD)}


def initial_dt(data, dx, dy, gamma=5.0 / 3.0, mu0=1.0):
    """Advective CFL surrogate (harness.py:105-116)."""
    rho = data[I_RHO]
    ax = np.abs(data[I_MX] / rho)
    ay = np.abs(data[I_MY] / rho)
    bsq = data[I_BX] ** 2 + data[I_BY] ** 2 + data[I_BZ] ** 2
    ekin = 0.5 * (data[I_MX] ** 2 + data[I_MY] ** 2 + data[I_MZ] ** 2) / rho
    pg = (gamma - 1.0) * (data[I_EN] - ekin - 0.5 * bsq / mu0)
    cf = np.sqrt(np.maximum(gamma * pg + bsq / mu0, 0.0) / rho)
    top = max(float(np.max(ax + cf)), float(np.max(ay + cf)), 1e-12)
    return 0.1 * min(dx, dy) / top


_HDR = "<4sIIIIddd"


def checkpoint_bytes(data, dx, dy, time):
    """Byte image of a reference checkpoint (mhd.py:250-257)."""
    nf, ny, nx = data.shape
    head = struct.pack(_HDR, b"XMHD", 1, nx, ny, nf, time, dx, dy)
    return head + b"".join(np.ascontiguousarray(data[k], dtype="<f8").tobytes()
                           for k in range(nf))
