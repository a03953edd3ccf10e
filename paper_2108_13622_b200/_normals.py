"""Parallel, value-exact ``Generator.standard_normal(n)`` on the run RNG's PCG64 stream.

The reference draws the power-iteration start vector as
``rng.standard_normal(n)`` from the run RNG (harness.py:130,164;
linearize.py:113).  At BASELINE configs 3/4 that is 134 M / 537 M normals, 1.4
/ 5.5 s on one host thread.  NumPy's normal sampler (a ziggurat) consumes one
raw 64-bit PCG64 output per normal most of the time and more on a rejection,
so the raw position where the k-th normal starts is only known after all
earlier normals were drawn.  This module splits the draw over host threads
without changing a single value:

* piece k (outputs [k*C, (k+1)*C)) is drawn by its own thread from a copy of
  the run generator advanced (``PCG64.advance``) to a raw position G_k a
  margin BEFORE the expected start k*C*(1+RHO) (RHO = mean extra raw draws
  per normal, measured);
* a sampler started a little early re-joins the true sequence of samples at
  the first raw position both visit (the sampler is a deterministic function
  of its raw position), so the true continuation of piece k-1 appears inside
  piece k's draw at some offset d_k: it is located by matching the L values
  piece k-1 drew past its end;
* a piece whose draw does not contain that continuation (the guess was late,
  or too early for its window) is redrawn sequentially from piece k-1's known
  start: slower, still exact;
* the run generator is left in the state a single ``standard_normal(n)``
  leaves it in (the last piece is short, so recomputing that state costs a
  short sequential draw).

``tests/test_host_cpu.py`` checks values and the stream continuation against a
plain ``standard_normal(n)``, including the fallback path.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

RHO = 0.0220          # mean extra raw PCG64 outputs per normal (measured: 0.02202 over 2e7)
RHO_VAR = 0.03        # variance bound of the extra raw outputs per normal (margin sizing)
L_MATCH = 8           # continuation values matched to align a piece
TAIL = 1 << 15        # length of the short last piece
MIN_PARALLEL = 1 << 21


def host_threads(cap=32):
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:   # pragma: no cover - non-Linux
        n = os.cpu_count() or 1
    return max(1, min(cap, n))


def _gen_at(state0, raw):
    """A generator on the same stream, ``raw`` PCG64 outputs further on."""
    bg = np.random.PCG64()
    bg.state = state0
    if raw:
        bg.advance(raw)
    return np.random.Generator(bg)


def _skip(gen, count, scratch):
    """Draw and discard ``count`` normals."""
    while count > 0:
        m = min(count, scratch.size)
        gen.standard_normal(out=scratch[:m])
        count -= m


def _plan(n, piece):
    """Piece sizes: full pieces of ``piece`` and a short last piece of TAIL values."""
    if n <= piece:
        return [n]
    sizes = [piece] * ((n - TAIL) // piece)
    rest = n - piece * len(sizes)
    while rest > TAIL:            # rest in (TAIL, piece + TAIL]
        m = rest - TAIL
        sizes.append(m)
        rest -= m
    sizes.append(rest)
    return sizes


class _Piece:
    __slots__ = ("start", "size", "guess", "window")

    def __init__(self, start, size, guess, window):
        self.start, self.size, self.guess, self.window = start, size, guess, window


def _pieces(n, piece, rho):
    out = []
    start = 0
    for k, size in enumerate(_plan(n, piece)):
        if k == 0:
            out.append(_Piece(0, size, 0, 0))
        else:
            expect = start * (1.0 + rho)
            margin = int(6.0 * math.sqrt(start * RHO_VAR)) + 2048
            guess = max(0, int(expect) - margin)
            out.append(_Piece(start, size, guess, 2 * margin + 4096))
        start += size
    return out


def draw(rng, n, alloc, sink, *, piece=1 << 21, threads=None, rho=RHO):
    """Draw ``rng.standard_normal(n)`` in parallel; hand the values to ``sink`` in order.

    ``alloc(m)`` returns a writable float64 NumPy array of at least m values (a
    page-locked buffer when the values go to a device); ``sink(i0, values)``
    receives outputs [i0, i0 + len(values)) in increasing order and returns an
    object with ``synchronize()`` (or None) that must complete before the
    buffer holding ``values`` is reused.  On return, ``rng`` is in the state a
    single ``rng.standard_normal(n)`` would have left it in.
    """
    bg = rng.bit_generator
    if not isinstance(bg, np.random.PCG64) or n < MIN_PARALLEL or (threads or host_threads()) < 2:
        buf = alloc(max(n, 1))[:n]
        rng.standard_normal(out=buf)
        ev = sink(0, buf)
        if ev is not None:
            ev.synchronize()
        return
    state0 = bg.state
    nthreads = threads or host_threads()
    plan = _pieces(n, piece, rho)
    nslots = min(len(plan), nthreads + 2)
    cap = max(p.size + p.window + L_MATCH for p in plan)
    slots = [alloc(cap) for _ in range(nslots)]
    released = [None] * nslots      # event guarding each slot's last upload

    def work(k):
        p = plan[k]
        slot = k % nslots
        ev = released[slot]
        if ev is not None:
            ev.synchronize()
        buf = slots[slot]
        m = p.size + p.window + (L_MATCH if k + 1 < len(plan) else 0)
        _gen_at(state0, p.guess).standard_normal(out=buf[:m])
        return buf

    scratch = np.empty(1 << 16)
    with ThreadPoolExecutor(max_workers=nthreads, thread_name_prefix="xmhd-normals") as pool:
        futs = {}
        nxt = 0

        def submit_upto(limit):
            nonlocal nxt
            while nxt < len(plan) and nxt < limit:
                futs[nxt] = pool.submit(work, nxt)
                nxt += 1

        submit_upto(nslots)
        cont = None
        src = (0, 0)            # (raw position, normals to skip) of the current piece's true start
        prev_src = None
        for k, p in enumerate(plan):
            buf = futs.pop(k).result()
            d = 0
            if k > 0:
                d = _locate(buf, p.window, cont)
                if d is None:   # redraw from piece k-1's known start
                    g = _gen_at(state0, prev_src[0])
                    _skip(g, prev_src[1] + plan[k - 1].size, scratch)
                    tail = L_MATCH if k + 1 < len(plan) else 0
                    g.standard_normal(out=buf[:p.size + tail])
                    src = (prev_src[0], prev_src[1] + plan[k - 1].size)
                    d = 0
                else:
                    src = (p.guess, d)
            vals = buf[d:d + p.size]
            if k + 1 < len(plan):
                cont = buf[d + p.size:d + p.size + L_MATCH].copy()
            released[k % nslots] = sink(p.start, vals)
            prev_src = src
            # the slot is handed to piece k + nslots only now (its worker waits on the event)
            submit_upto(k + 1 + nslots)
        for ev in released:
            if ev is not None:
                ev.synchronize()

    # the run generator's state after exactly n normals
    g = _gen_at(state0, src[0])
    _skip(g, src[1] + plan[-1].size, scratch)
    st = g.bit_generator.state
    st["has_uint32"] = state0["has_uint32"]
    st["uinteger"] = state0["uinteger"]
    bg.state = st


def _locate(buf, window, cont):
    """Offset d in [0, window] with buf[d:d+L] == cont, or None."""
    head = buf[:window + 1]
    for d in np.flatnonzero(head == cont[0]):
        d = int(d)
        if np.array_equal(buf[d:d + L_MATCH], cont):
            return d
    return None


def standard_normal(rng, n, **kw):
    """``rng.standard_normal(n)`` drawn in parallel (same values, same stream state)."""
    out = np.empty(n)

    def sink(i0, vals):
        out[i0:i0 + vals.size] = vals
        return None

    draw(rng, n, np.empty, sink, **kw)
    return out
