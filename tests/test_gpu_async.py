"""Asynchronous steps and the one-launch Leja loop against the synchronous paths.

The asynchronous step (integrators._step_async) enqueues a whole exponential
step and reads one record; the Leja loop runs every Newton term of a
phi-action inside one cooperative launch.  Both must be invisible to the
reference's semantics: the same bits, counters, step sequence and cache
state as the per-call synchronous driver (and hence the reference, which
test_gpu_parity pins), including the mid-step events that force a replay.
"""

import contextlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@contextlib.contextmanager
def mode(async_on=True, loop=True, tile=True):
    """loop: phi-actions as one launch (tile: the 2D-tile loop, else the
    sliding-window kernel in a loop); not loop: one launch per Newton term."""
    from paper_2108_13622_b200 import _lib, integrators, leja, mhd
    old = (integrators.ASYNC, leja.LOOP_MAX_CELLS)
    integrators.ASYNC = async_on
    leja.LOOP_MAX_CELLS = (1 << 20) if loop else 0

    def reset(kind):
        for c in mhd._ctx_cache.values():
            c.loop_ok = None
            _lib.load().xmhd_set_loop_kind(c.h, kind)
    reset(0 if tile else 1)
    try:
        yield
    finally:
        integrators.ASYNC, leja.LOOP_MAX_CELLS = old
        reset(0)


def _run(setup, scheme, tol):
    import paper_2108_13622_b200 as xb
    from paper_2108_13622_b200 import leja
    leja._coeff_cache.clear()
    rep = xb.run(xb.RunConfig(scenario=setup, scheme=scheme, tol=tol))
    steps = [(s.dt, s.error, s.rhs_calls, s.phi_iterations, s.phi_applications, s.accepted)
             for s in rep.steps]
    return rep, steps, list(leja._coeff_cache)


@pytest.mark.parametrize("which", ["kh", "harris"])
def test_async_run_is_bitwise_the_synchronous_run(which):
    import paper_2108_13622_b200 as xb
    from paper_2108_13622_b200 import integrators, scenarios as sc
    if which == "kh":
        setup, scheme, tol = sc.kh_setup(32, t_final=0.15), xb.Scheme.EXPRB43, 1e-4
    else:
        setup, scheme, tol = sc.harris_setup(32, t_final=0.6), xb.Scheme.EXPRB54S4, 1e-6
    _run(setup, scheme, tol)                    # contexts exist before the modes switch
    with mode(async_on=False, loop=False):      # per-term launches, host batches
        ref, ref_steps, ref_keys = _run(setup, scheme, tol)
    with mode(async_on=False, loop=True, tile=False):   # sliding-window loop, one launch
        sl, sl_steps, sl_keys = _run(setup, scheme, tol)
    with mode(async_on=False, loop=True):       # 2D-tile loop, one launch per phi-action
        lp, lp_steps, lp_keys = _run(setup, scheme, tol)
    r0 = integrators.replays
    with mode(async_on=True, loop=True):        # the same, one host wait per step
        asy, asy_steps, asy_keys = _run(setup, scheme, tol)
    assert ref.accepted >= 3
    assert integrators.replays == r0      # nothing in these runs needs a replay
    # same kernel body and reduction order: bitwise
    for other, steps, keys, base in ((sl, sl_steps, sl_keys, (ref, ref_steps, ref_keys)),
                                     (asy, asy_steps, asy_keys, (lp, lp_steps, lp_keys))):
        b, b_steps, b_keys = base
        assert steps == b_steps
        assert keys == b_keys
        assert (other.rhs_evals, other.phi_iterations) == (b.rhs_evals, b.phi_iterations)
        assert other.checksum == b.checksum
    # tiles sum the norms in another (fixed) order, the kind of difference the
    # reference's own BLAS thread count makes: the north-star bar for adaptive
    # runs (same accepted/rejected sequence and counters, final state 1e-8)
    assert [s[2:] for s in lp_steps] == [s[2:] for s in ref_steps]
    assert np.allclose([s[0] for s in lp_steps], [s[0] for s in ref_steps], rtol=1e-6, atol=0)
    assert (lp.rhs_evals, lp.phi_iterations) == (ref.rhs_evals, ref.phi_iterations)
    a = lp.final_state.flat().cpu().numpy()
    b = ref.final_state.flat().cpu().numpy()
    assert np.linalg.norm(a - b) <= 1e-8 * np.linalg.norm(b)


def _lin(n=24, seed=4):
    import paper_2108_13622_b200 as xb
    from paper_2108_13622_b200 import scenarios as sc
    s = sc.kh_setup(n)
    q = sc.initial_fields(s)
    q = q + 1e-3 * np.random.default_rng(seed).standard_normal(q.shape)
    st = xb.StateGrid(n, n, s.dx, s.dy, torch.from_numpy(q).cuda())
    op = xb.RhsOperator(xb.MhdRhs(st, xb.MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa)))
    return xb, st, op


def _same(a, b):
    assert a.converged == b.converged
    assert a.rhs_calls == b.rhs_calls
    assert a.phi_iterations == b.phi_iterations
    assert a.phi_applications == b.phi_applications
    assert (a.error_estimate == b.error_estimate or
            (np.isnan(a.error_estimate) and np.isnan(b.error_estimate)))
    assert torch.equal(a.new_state, b.new_state)


def test_async_step_replays_on_nonfinite_rhs():
    """A stage that overflows makes F non-finite: the reference raises
    RhsBlowupError mid-step and stops calling F; the asynchronous step sees
    the flag in its record and replays synchronously (same counters)."""
    from paper_2108_13622_b200 import integrators
    xb, st, op = _lin()
    u = st.flat()
    res = {}
    for async_on in (False, True):
        with mode(async_on=async_on):
            lin = xb.FrozenLinearization(op, u)
            r0 = integrators.replays
            res[async_on] = xb.step(xb.Scheme.EXPRB43, op, u, 1e300, alpha=0.0, tol=1e-4,
                                    lin=lin)
            if async_on:
                assert integrators.replays == r0 + 1
    assert not res[True].converged and res[True].error_estimate == np.inf
    _same(res[True], res[False])


def test_async_step_replays_when_a_phi_action_needs_a_second_chunk():
    """A step whose phi-actions pass 64 Newton terms: the device loop stops at
    the end of the first chunk, the record shows it, the step is replayed with
    the reference's chunk growth and cache updates."""
    from paper_2108_13622_b200 import integrators, leja
    xb, st, op = _lin()
    u = st.flat()
    lin0 = xb.FrozenLinearization(op, u)
    alpha = xb.estimate_alpha(lin0, None, rng=np.random.default_rng(0)).alpha
    dt = 60.0 / alpha
    res, keys = {}, {}
    for async_on in (False, True):
        with mode(async_on=async_on):
            leja._coeff_cache.clear()
            lin = xb.FrozenLinearization(op, u)
            r0 = integrators.replays
            res[async_on] = xb.step(xb.Scheme.EXPRB43, op, u, dt, alpha=alpha, tol=1e-6, lin=lin)
            keys[async_on] = [(k, v.size) for k, v in leja._coeff_cache.items()]
            if async_on:
                assert integrators.replays == r0 + 1
    assert res[False].phi_iterations > 64
    _same(res[True], res[False])
    assert keys[True] == keys[False]


@pytest.mark.parametrize("n", [40, 37])
def test_loop_kernels_against_per_term_launches(n):
    """One cooperative launch per phi-action vs one launch per Newton term,
    across a coefficient-chunk growth (degree > 64): the sliding-window loop
    is bitwise the per-term path; the 2D-tile loop (partial tiles when
    n = 37) matches it within the norm-order rounding floor at low degree and
    with the same degree at high degree, and matches the NumPy oracle."""
    from oracle import leja_np as olj, mhd_np
    from paper_2108_13622_b200 import leja
    xb, st, op = _lin(n=n)
    lin = xb.FrozenLinearization(op, st.flat())
    alpha = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0)).alpha
    v = torch.from_numpy(np.random.default_rng(9).standard_normal(st.flat().numel())).cuda()
    out = {}
    for key, kw in (("batch", dict(loop=False)), ("slide", dict(loop=True, tile=False)),
                    ("tile", dict(loop=True, tile=True))):
        with mode(**kw):
            leja._coeff_cache.clear()
            for adt in (3.0, 80.0):
                sh = xb.shift_and_scale(adt)
                c = op.calls
                r = xb.apply_phi_leja(1, xb.JacobianAction(lin), v, adt / alpha, sh, 1e-10)
                out[(key, adt)] = (r, op.calls - c)
    for adt in (3.0, 80.0):
        (a, ca), (b, cb) = out[("batch", adt)], out[("slide", adt)]
        assert (a.iterations, a.converged, a.residual, ca) == (b.iterations, b.converged,
                                                               b.residual, cb)
        assert torch.equal(a.vector, b.vector)
        (t, ct) = out[("tile", adt)]
        assert (t.iterations, t.converged, ct) == (a.iterations, a.converged, ca)
    assert out[("tile", 80.0)][0].iterations > 64
    t, a = out[("tile", 3.0)][0], out[("batch", 3.0)][0]
    assert (t.vector - a.vector).norm() <= 1e-12 * a.vector.norm()
    # the tile loop against the oracle (the reference's algorithm) at low degree
    s = st
    q = s.data.cpu().numpy()
    prm = op.fn.params

    def f(flat):
        return mhd_np.rhs(flat.reshape(q.shape), s.dx, s.dy, prm.mu, prm.eta, prm.kappa)
    olin = olj.Frozen(olj.CountedRhs(f), q.reshape(-1))
    sh = xb.shift_and_scale(3.0)
    ref = olj.phi_leja(1, lambda x: olj.fd_jvp(olin, x), v.cpu().numpy(), 3.0 / alpha, sh.q,
                       sh.theta, 1e-10, olj.CoeffCache())
    assert t.iterations == ref.iterations
    assert np.linalg.norm(t.vector.cpu().numpy() - ref.vector) <= 1e-10 * np.linalg.norm(ref.vector)


def test_batched_driver_when_a_batch_ends_at_a_chunk_boundary():
    """Host-paced batches (large grids): a batch that ends exactly at term 63
    leaves the device at the end of the first coefficient chunk; the driver
    must extend the table and continue, like the reference's growth."""
    from paper_2108_13622_b200 import leja
    xb, st, op = _lin(n=40)
    lin = xb.FrozenLinearization(op, st.flat())
    alpha = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0)).alpha
    v = torch.from_numpy(np.random.default_rng(9).standard_normal(st.flat().numel())).cuda()
    adt = 80.0
    sh = xb.shift_and_scale(adt)
    out = {}
    for key, kw in (("loop", dict(loop=True, tile=False)), ("batch", dict(loop=False))):
        with mode(**kw):
            leja._coeff_cache.clear()
            leja._degree_hint.clear()
            if key == "batch":
                theta = sh.theta
                leja._degree_hint[(1, int(round(4.0 * np.log2(theta))))] = 63
            out[key] = xb.apply_phi_leja(1, xb.JacobianAction(lin), v, adt / alpha, sh, 1e-10)
    a, b = out["loop"], out["batch"]
    assert a.iterations > 64 and a.iterations == b.iterations and a.converged == b.converged
    assert torch.equal(a.vector, b.vector)


@pytest.mark.parametrize("kw", [dict(loop=False), dict(loop=True, tile=False),
                                dict(loop=True, tile=True)], ids=["batch", "slide", "tile"])
def test_deferred_interpolant_stores_are_bitwise(kw):
    """Every other Newton term keeps p' in registers and the next term stores
    both additions in the reference's order: the interpolant, the residuals
    and the iteration counts are bitwise those of a store per term, for
    converged calls ending on either parity, a chunk growth, and a blow-up
    (which returns the interpolant before the failing term)."""
    from paper_2108_13622_b200 import _lib, leja, mhd
    xb, st, op = _lin(n=40)
    lin = xb.FrozenLinearization(op, st.flat())
    alpha = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0)).alpha
    v = torch.from_numpy(np.random.default_rng(9).standard_normal(st.flat().numel())).cuda()
    cases = [(1, 1.0, 1.0), (1, 3.0, 1.0), (3, 7.0, 1.0), (1, 80.0, 1.0), (1, 50.0, 1e-3)]
    out = {}
    try:
        for defer in (0, 1):
            for c in mhd._ctx_cache.values():
                _lib.load().xmhd_set_leja_defer(c.h, defer)
            with mode(**kw):
                for l, adt, shrink in cases:
                    leja._coeff_cache.clear()
                    sh = xb.shift_and_scale(shrink * adt)
                    r = xb.apply_phi_leja(l, xb.JacobianAction(lin), v, adt / alpha, sh, 1e-10)
                    out[(defer, l, adt, shrink)] = r
    finally:
        for c in mhd._ctx_cache.values():
            _lib.load().xmhd_set_leja_defer(c.h, 1)
    parities = set()
    for l, adt, shrink in cases:
        a, b = out[(0, l, adt, shrink)], out[(1, l, adt, shrink)]
        assert (a.iterations, a.converged, a.residual) == (b.iterations, b.converged, b.residual)
        assert torch.equal(a.vector, b.vector)
        if a.converged:
            parities.add(a.iterations % 2)
    assert parities == {0, 1}
    assert not out[(1, 1, 50.0, 1e-3)].converged          # blow-up case
    assert out[(1, 1, 80.0, 1.0)].iterations > 64          # chunk growth


@pytest.mark.parametrize("which", ["kh", "harris"])
def test_native_step_is_bitwise_the_python_issued_step(which):
    """xmhd_step_async (csrc/steps.cpp) enqueues the operations of
    _step_exprb43 / _step_exprb54s4 in the same order: the same run bit for
    bit as the asynchronous step issued from Python."""
    import paper_2108_13622_b200 as xb
    from paper_2108_13622_b200 import integrators, scenarios as sc
    if which == "kh":
        setup, scheme, tol = sc.kh_setup(32, t_final=0.15), xb.Scheme.EXPRB43, 1e-4
    else:
        setup, scheme, tol = sc.harris_setup(32, t_final=0.6), xb.Scheme.EXPRB54S4, 1e-6
    out = {}
    old = integrators.NATIVE_STEP
    try:
        for native in (False, True):
            integrators.NATIVE_STEP = native
            with mode(async_on=True, loop=True):
                out[native] = _run(setup, scheme, tol)
    finally:
        integrators.NATIVE_STEP = old
    (a, sa, ka), (b, sb, kb) = out[False], out[True]
    assert sa == sb and ka == kb
    assert (a.rhs_evals, a.phi_iterations, a.checksum) == (b.rhs_evals, b.phi_iterations,
                                                           b.checksum)


def test_deferred_linearization_raises_like_the_constructor():
    """FrozenLinearization with a known ||u|| enqueues F(u) without waiting;
    a non-finite F(u) raises the reference's RhsBlowupError (same message and
    cells) from check(), from estimate_alpha and from step()."""
    xb, st, op = _lin(n=24)
    u = st.flat().clone()
    u[5 * 24 * 24 + 7] = float("nan")
    with pytest.raises(xb.RhsBlowupError) as eager:
        xb.FrozenLinearization(op, u)
    for use in ("check", "alpha", "step"):
        lin = xb.FrozenLinearization(op, u, base_norm=1.0)
        with pytest.raises(xb.RhsBlowupError) as lazy:
            if use == "check":
                lin.check()
            elif use == "alpha":
                xb.estimate_alpha(lin, None, rng=np.random.default_rng(0))
            else:
                xb.step(xb.Scheme.EXPRB43, op, u, 1e-3, alpha=10.0, tol=1e-4, lin=lin)
        assert str(lazy.value) == str(eager.value)
        assert lazy.value.cells == eager.value.cells


def test_lazy_divb_and_norm_match_the_eager_run():
    """The harness's deferred div B log and carried state norm give the run
    of the eager path (div B read every step, ||u|| reduced by the
    linearization): same report, same bits."""
    import paper_2108_13622_b200 as xb
    from paper_2108_13622_b200 import harness, scenarios as sc
    setup = sc.kh_setup(32, t_final=0.15)
    lazy = xb.run(xb.RunConfig(scenario=setup, tol=1e-4))
    old = harness._Domain.divb_async_ok
    try:
        harness._Domain.divb_async_ok = False
        eager = xb.run(xb.RunConfig(scenario=setup, tol=1e-4))
    finally:
        harness._Domain.divb_async_ok = old
    assert lazy.max_divb == eager.max_divb
    assert lazy.checksum == eager.checksum and lazy.rhs_evals == eager.rhs_evals
