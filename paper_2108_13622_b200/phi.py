"""phi-function divided differences for the Leja Newton coefficients.

Host mirror of the parts of ``pkg/src/xmhd/phi.py`` that feed the hot path:
``_phi_divided_diffs`` (phi.py:99-144) runs in the native library's C++ port
(``csrc/divdiff.cpp``, bitwise equal to the NumPy routine), and
``divided_differences`` / ``phi_scalar`` keep the reference signatures.
``phi_dense`` (the dense-matrix oracle of phi.py:63-88) is out of the hot path
and lives only in the test oracle.
"""

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from paper_2108_13622_b200 import _lib

MAX_ORDER = 4            # phi.py:15
_SERIES_SWITCH = 0.5     # phi.py:24


def _check_order(l):
    if not isinstance(l, (int, np.integer)) or l < 0 or l > MAX_ORDER:
        raise ValueError(f"phi order must be an integer in [0, {MAX_ORDER}], got {l!r}")


def phi_scalar(l, z):
    """phi_l(z) for a real or complex scalar (phi.py:32-47)."""
    _check_order(l)
    if abs(z) >= _SERIES_SWITCH:
        # upward recursion phi_{j+1} = (phi_j - 1/j!) / z from phi_0 = exp
        out = np.exp(z)
        for j in range(l):
            out = (out - 1.0 / math.factorial(j)) / z
        return out
    # small |z|: direct series sum_k z^k / (k+l)!, cancellation-free
    acc = term = 1.0 / math.factorial(l)
    k = 1
    while k < 64:
        term = term * z / (k + l)
        acc = acc + term
        if abs(term) <= 1e-16 * abs(acc):
            break
        k += 1
    return acc


def _phi_divided_diffs(l, nodes, subdiag=1.0):
    """First column of phi_l of the lower-bidiagonal node matrix (phi.py:99-144), native."""
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    out = np.empty(nodes.size)
    rc = _lib.load().xmhd_phi_divided_diffs(
        int(l), nodes.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(nodes.size),
        float(subdiag), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if rc != _lib.OK:
        raise ValueError("xmhd_phi_divided_diffs rejected its arguments")
    return out


@dataclass(frozen=True)
class DividedDiffTable:
    """Newton divided differences of phi_l at a node sequence (phi.py:91-96)."""
    nodes: np.ndarray
    coeffs: np.ndarray
    order: int


def divided_differences(l, nodes):
    """Newton divided differences of phi_l at real nodes (phi.py:147-161)."""
    _check_order(l)
    nodes = np.asarray(nodes, dtype=float)
    if nodes.ndim != 1 or nodes.size == 0:
        raise ValueError("divided_differences requires a nonempty 1-d node sequence")
    if nodes.size > 512:
        raise ValueError("node sequence longer than the 512-node oracle scale")
    return DividedDiffTable(nodes=nodes, coeffs=_phi_divided_diffs(l, nodes, 1.0), order=l)


def newton_eval(table, z):
    """Horner evaluation of a DividedDiffTable's Newton form at z (phi.py:164-170)."""
    x = table.nodes
    result = np.full_like(np.asarray(z, dtype=float), table.coeffs[-1])
    for k in range(x.size - 2, -1, -1):
        result = result * (z - x[k]) + table.coeffs[k]
    return result
