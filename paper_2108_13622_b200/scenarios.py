"""Seeded initial states for the BASELINE.json configurations 0-4.

The reference's presets (``pkg/src/xmhd/scenarios.py:75-194``) use other
domains, ICs and boundary conditions, so the BASELINE configs need their own
initializers (SURVEY.md §0 finding 4, §8(d)).  They sample closed-form fields
at cell centres ``x_min + (i + 1/2) dx`` like ``scenarios.py:59-62`` and form
the total energy from the pressure closure like ``scenarios.py:165-166``.
These are host-side input builders (NumPy); everything that acts on the state
afterwards runs on the device.

Configs (BASELINE.json ``configs``):

0. Kelvin-Helmholtz 128^2 on [0,1) x [-1,1), EXPRB43, tol 1e-4, t_end 0.5.
1. Config-0 state at 2048^2 + 1e-2 x seeded sum of 16 random-phase Fourier
   modes per field (|k| <= 8); v a seeded unit Gaussian vector; phi_1 sweep.
2. Double Harris sheet 512^2 on [0,25.6) x [-12.8,12.8), EXPRB54s4, tol 1e-6,
   t_end 10.
3. Config 0 at 4096^2, tol 1e-5, 20 adaptive steps.
4. Config 2 at 8192^2 (and 16384^2), eta 1e-3, tol 1e-6, 10 adaptive steps.
"""

from dataclasses import dataclass, field

import numpy as np

NFIELD = 8
RHO, MX, MY, MZ, BX, BY, BZ, EN = range(NFIELD)


@dataclass
class Setup:
    """A runnable configuration: geometry, physics, scheme and stopping rule."""
    name: str
    nx: int
    ny: int
    x_min: float
    x_max: float
    y_min: float
    y_max: float
    mu: float
    eta: float
    kappa: float
    gamma: float = 5.0 / 3.0
    mu0: float = 1.0
    scheme: str = "exprb43"
    tol: float = 1e-4
    t_final: float = 0.5
    max_accepted: int | None = None
    seed: int = 0
    kind: str = "kh"
    extra: dict = field(default_factory=dict)

    @property
    def dx(self):
        return (self.x_max - self.x_min) / self.nx

    @property
    def dy(self):
        return (self.y_max - self.y_min) / self.ny

    def centres(self, rows=None):
        """Cell-centre meshgrid of all rows, or of rows [y0, y1) (a y-strip)."""
        y0, y1 = (0, self.ny) if rows is None else rows
        x = self.x_min + (np.arange(self.nx) + 0.5) * self.dx
        y = self.y_min + (np.arange(y0, y1) + 0.5) * self.dy
        return np.meshgrid(x, y)


def kh_setup(n=128, tol=1e-4, t_final=0.5, max_accepted=None, seed=0, name="C0"):
    return Setup(name=name, nx=n, ny=n, x_min=0.0, x_max=1.0, y_min=-1.0, y_max=1.0,
                 mu=1e-3, eta=1e-3, kappa=1e-3, scheme="exprb43", tol=tol,
                 t_final=t_final, max_accepted=max_accepted, seed=seed, kind="kh")


def harris_setup(n=512, eta=5e-3, tol=1e-6, t_final=10.0, max_accepted=None, seed=0,
                 name="C2"):
    return Setup(name=name, nx=n, ny=n, x_min=0.0, x_max=25.6, y_min=-12.8, y_max=12.8,
                 mu=1e-3, eta=eta, kappa=1e-3, scheme="exprb54s4", tol=tol,
                 t_final=t_final, max_accepted=max_accepted, seed=seed, kind="harris")


CONFIGS = {
    0: lambda: kh_setup(128, name="C0"),
    1: lambda: Setup(**{**kh_setup(2048).__dict__, "name": "C1", "kind": "kh-modes",
                        "extra": {"mode_seed": 1, "v_seed": 2}}),
    2: lambda: harris_setup(512, name="C2"),
    3: lambda: kh_setup(4096, tol=1e-5, t_final=1e9, max_accepted=20, name="C3"),
    4: lambda: harris_setup(8192, eta=1e-3, tol=1e-6, t_final=1e9, max_accepted=10,
                            name="C4"),
    # config 4's weak-scaling case: 16384^2 across 8 GPUs (17.2 GB per state vector)
    "4w": lambda: harris_setup(16384, eta=1e-3, tol=1e-6, t_final=1e9, max_accepted=10,
                               name="C4w"),
}


def _noise_rows(seed, nx, y0, y1):
    """Rows [y0, y1) of default_rng(seed).uniform(-1, 1, size=(ny, nx)): a
    uniform double takes exactly one raw PCG64 output, so the rows start
    y0*nx outputs into the stream (PCG64.advance) -- bitwise the same values."""
    bg = np.random.default_rng(seed).bit_generator
    bg.advance(y0 * nx)
    return np.random.Generator(bg).uniform(-1.0, 1.0, size=(y1 - y0, nx))


def kh_fields(s, rows=None):
    """Config 0: tanh shear pair, seeded vy noise in the shear envelopes."""
    y0, y1 = (0, s.ny) if rows is None else rows
    x, y = s.centres(rows)
    ny = y1 - y0
    vx = 0.5 * (np.tanh((y + 0.5) / 0.05) - np.tanh((y - 0.5) / 0.05) - 1.0)
    if rows is None:
        noise = np.random.default_rng(s.seed).uniform(-1.0, 1.0, size=(s.ny, s.nx))
    else:
        noise = _noise_rows(s.seed, s.nx, y0, y1)
    vy = 1e-3 * noise * np.exp(-((np.abs(y) - 0.5) / 0.1) ** 2)
    rho = np.ones((ny, s.nx))
    pres = np.ones((ny, s.nx))
    bx = 0.1
    q = np.zeros((NFIELD, ny, s.nx))
    q[RHO] = rho
    q[MX] = rho * vx
    q[MY] = rho * vy
    q[BX] = bx
    q[EN] = (pres / (s.gamma - 1.0) + 0.5 * rho * (vx ** 2 + vy ** 2)
             + 0.5 * bx ** 2 / s.mu0)
    return q


def fourier_modes(s, amplitude=1e-2, modes=16, kmax=8, seed=None, rows=None):
    """Seeded smooth field per conserved variable: sum of random-phase modes."""
    rng = np.random.default_rng(s.seed if seed is None else seed)
    x, y = s.centres(rows)
    lx = s.x_max - s.x_min
    ly = s.y_max - s.y_min
    xs = (x - s.x_min) / lx
    ys = (y - s.y_min) / ly
    out = np.zeros((NFIELD,) + x.shape)
    for f in range(NFIELD):
        k = 0
        while k < modes:
            kx, ky = rng.integers(-kmax, kmax + 1, size=2)
            if not 1 <= kx * kx + ky * ky <= kmax * kmax:
                continue
            ph = rng.uniform(0.0, 2.0 * np.pi)
            out[f] += np.cos(2.0 * np.pi * (kx * xs + ky * ys) + ph)
            k += 1
    return amplitude * out


def harris_fields(s, rows=None):
    """Config 2: double Harris sheet with a curl(psi z) flux perturbation."""
    x, y = s.centres(rows)
    w = 0.5
    bx0 = np.tanh((y + 6.4) / w) - np.tanh((y - 6.4) / w) - 1.0
    rho = 1.0 + 1.0 / np.cosh((y + 6.4) / w) ** 2 + 1.0 / np.cosh((y - 6.4) / w) ** 2
    pres = 0.5 * (1.0 + rho - bx0 ** 2)
    lx, ly = 25.6, 12.8
    kx, ky = 2.0 * np.pi / lx, 2.0 * np.pi / ly
    psi0 = 0.1
    # dB = curl(psi z) = (d psi / dy, -d psi / dx)
    dbx = -psi0 * ky * np.cos(kx * x) * np.sin(ky * y)
    dby = psi0 * kx * np.sin(kx * x) * np.cos(ky * y)
    bx = bx0 + dbx
    by = dby
    q = np.zeros((NFIELD,) + x.shape)
    q[RHO] = rho
    q[BX] = bx
    q[BY] = by
    q[EN] = pres / (s.gamma - 1.0) + 0.5 * (bx ** 2 + by ** 2) / s.mu0
    return q


def initial_fields(s, rows=None):
    """(8, ny, nx) float64 initial conserved state of a Setup, or only its rows
    [y0, y1) (a y-strip builds its own rows: bitwise those of the full state)."""
    if s.kind == "kh":
        return kh_fields(s, rows)
    if s.kind == "kh-modes":
        return kh_fields(s, rows) + fourier_modes(s, seed=s.extra.get("mode_seed", 1), rows=rows)
    if s.kind == "harris":
        return harris_fields(s, rows)
    raise ValueError(f"unknown setup kind {s.kind!r}")


def unit_gaussian(n, seed):
    """Seeded unit-norm Gaussian vector (config 1's v).

    Normalised with NumPy's pairwise ``add.reduce`` rather than
    ``np.linalg.norm``: OpenBLAS ``ddot`` splits large vectors over threads, so
    its last bit depends on the host's core count, and the committed golden
    fixtures (tests/golden/large/) must see the same v on every host."""
    v = np.random.default_rng(seed).standard_normal(n)
    return v / np.sqrt(np.add.reduce(v * v))
