"""CPU-side checks: the C-ABI library builds, loads and exports every declared
symbol; the host logic around the kernels (coefficients, Leja points,
controllers) matches the reference's golden vectors.  No device compute here."""

import os
import re

import numpy as np
import pytest
import torch

import golden_io

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2108_13622_b200 import _lib
    return _lib.load()


def header_functions():
    text = open(os.path.join(REPO, "include", "xmhd_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|long long|const char\*)\s+(xmhd_\w+)\s*\(",
                                 text, flags=re.M)))


def test_library_exports_every_declared_symbol(lib):
    from paper_2108_13622_b200 import _lib
    names = header_functions()
    assert len(names) >= 25
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.EXPORTED)


def test_library_is_sm100a(lib):
    import subprocess
    from paper_2108_13622_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.library_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_native_divided_differences_bitwise(lib):
    from paper_2108_13622_b200 import leja, phi
    g = golden_io.arrays("coeff_cases")
    nodes = leja.leja_points(64)
    for l in (0, 1, 3):
        assert np.array_equal(phi.divided_differences(l, nodes).coeffs, g[f"divdiff_l{l}"])


def test_newton_coefficients_bitwise(lib):
    from paper_2108_13622_b200 import leja
    g = golden_io.arrays("coeff_cases")
    for m in golden_io.meta()["coeff"]:
        leja._coeff_cache.clear()
        c = leja._newton_coeffs(m["l"], m["q"], m["theta"], m["count"])
        assert np.array_equal(c, g[m["key"]]), m["key"]


def test_coefficient_cache_contract(lib):
    from paper_2108_13622_b200 import leja
    leja._coeff_cache.clear()
    big = leja._newton_coeffs(1, -5.0, 2.5, 256)
    assert leja._newton_coeffs(1, -5.0, 2.5, 64) is big
    for k in range(70):
        leja._newton_coeffs(0, -1.0 - k, 0.5 + k, 64)
    assert len(leja._coeff_cache) == 65
    assert (1, -5.0, 2.5) not in leja._coeff_cache


def test_leja_points_bitwise():
    from paper_2108_13622_b200 import leja
    g = golden_io.arrays("coeff_cases")
    assert np.array_equal(leja.leja_points(500), g["leja_points"])
    assert leja.leja_points(1)[0] == 2.0
    with pytest.raises(ValueError):
        leja.leja_points(0)
    with pytest.raises(ValueError):
        leja.leja_points(501)


def test_shift_and_scale():
    from paper_2108_13622_b200 import shift_and_scale
    s = shift_and_scale(4.0)
    assert s.q == -2.0 and s.theta == 1.0
    with pytest.raises(ValueError):
        shift_and_scale(0.0)


def test_controllers_worked_examples():
    import math
    from paper_2108_13622_b200 import controllers as c
    k = c.ControllerConstants()
    assert abs(c.cost_next(0.1, 0.05, 100.0, 100.0, k) - 0.1 * 1.37412002) <= 1e-12
    assert abs(c.cost_next(0.1, 0.05, 200.0, 100.0, k) - 0.1 * 0.64446017) <= 1e-12
    delta = (math.log(1e6) - math.log(1.0)) / (math.log(0.1) - math.log(0.2))
    s = math.exp(-0.65241444 * math.tanh(0.26862269 * delta))
    assert abs(c.cost_next(0.1, 0.2, 1e6, 1.0, k) - 0.1 * s) <= 1e-12
    assert c.traditional_next(0.1, 0.0, 1e-4, 3) == 0.2
    assert c.combine(1.0, 2.0) == 1.0 and c.accept(1e-4, 1e-4)


def test_controllers_match_oracle():
    from oracle import steppers_np as st
    from paper_2108_13622_b200 import controllers as c
    rng = np.random.default_rng(1)
    for _ in range(200):
        dt, dtp = rng.uniform(1e-4, 1e-1, 2)
        cost, costp = rng.uniform(1.0, 1e4, 2)
        err, tol = 10.0 ** rng.uniform(-9, -2), 10.0 ** rng.uniform(-8, -3)
        p = int(rng.integers(1, 5))
        assert c.cost_next(dt, dtp, cost, costp) == st.cost_next(dt, dtp, cost, costp)
        assert c.traditional_next(dt, err, tol, p) == st.trad_next(dt, err, tol, p)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_compute_without_gpu_fails_loudly():
    import paper_2108_13622_b200 as xb
    st = xb.StateGrid.zeros(4, 4, 0.1, 0.1)
    with pytest.raises(xb.NativeUnavailable):
        xb.mhd_rhs(st, xb.MHDParams(0.0, 0.0, 0.0))


def test_newton_coeffs_many_matches_sequential_calls(lib):
    """The batched coefficient lookup (concurrent misses) leaves the cache and
    returns the tables exactly as one _newton_coeffs call per key would,
    including repeated keys and FIFO eviction at 65 entries."""
    import numpy as np
    from paper_2108_13622_b200 import leja
    keys = [(1, -0.5 * a, 0.25 * a) for a in np.linspace(0.3, 9.0, 70)]
    keys = keys[:3] + [keys[1]] + keys[3:] + [keys[0]]
    leja._coeff_cache.clear()
    ref = [leja._newton_coeffs(*k, 64) for k in keys]
    ref_keys = list(leja._coeff_cache)
    leja._coeff_cache.clear()
    got = leja.newton_coeffs_many(keys, 64)
    assert list(leja._coeff_cache) == ref_keys
    assert all(np.array_equal(a, b) for a, b in zip(ref, got))
    leja._coeff_cache.clear()


def test_prefetched_start_vector_is_the_run_rng_stream():
    """The run RNG's first standard_normal(n) is drawn ahead on a host thread
    (into page-locked memory when CUDA is up); values and the continuation of
    the stream equal the reference's plain draws (harness.py:130,
    linearize.py:113)."""
    from paper_2108_13622_b200 import harness
    n = 100_003
    pre = harness._PrefetchedNormals(11, n)
    ref = np.random.default_rng(11)
    assert np.array_equal(pre.standard_normal(n), ref.standard_normal(n))
    assert np.array_equal(pre.standard_normal(7), ref.standard_normal(7))


@pytest.mark.parametrize("n,piece,rho", [
    (3_000_017, 1 << 17, None),     # 23 pieces aligned on their continuation
    (2_500_000, 1 << 16, 0.05),     # guesses too late: every piece redrawn from its predecessor
    (2_200_000, 1 << 16, 0.0),      # guesses early beyond the window: redrawn as well
    (1 << 21, 1 << 21, None),       # one piece
    (1_000_003, 1 << 16, None),     # below the parallel threshold: one plain draw
])
def test_parallel_normals_equal_one_draw(n, piece, rho):
    """The start vector drawn in parallel pieces (``_normals.draw``) is value
    for value the reference's single ``rng.standard_normal(n)``
    (harness.py:130, linearize.py:113) and leaves the run RNG in the same
    state, including when a piece's alignment falls back to a redraw."""
    from paper_2108_13622_b200 import _normals
    kw = {} if rho is None else {"rho": rho}
    r1, r2 = np.random.default_rng(7), np.random.default_rng(7)
    got = _normals.standard_normal(r1, n, piece=piece, threads=4, **kw)
    assert np.array_equal(got, r2.standard_normal(n))
    assert r1.bit_generator.state == r2.bit_generator.state
    assert np.array_equal(r1.standard_normal(5), r2.standard_normal(5))
