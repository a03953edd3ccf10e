"""y-strip domain decomposition of the hot path over ranks.

Partitioning: contiguous y-strips — rank r owns rows [y0, y0+ny_r) of every
field with the full x extent, so x-periodicity stays rank-local ("row bands",
SPEC.md:486).  Per stencil evaluation a rank needs 2 ghost rows of the state
from each y-neighbour (the ±2 footprint of mhd.py:143,222-223); the periodic
wrap connects rank 0 and rank P-1, a reflecting wall makes the edge rank build
its own mirrored ghost rows (mhd.py:77-105).

Per Leja term (leja.py:133-148) the driver below enqueues, without any host
synchronisation:

    pack the boundary rows of the current y          (device kernel)
    2-row halo exchange with both y-neighbours        (torch.distributed P2P: NCCL/NVLink)
    fused FD-JVP + Newton term on the strip           (stencil kernel, BC_HALO rows)
    allreduce of [sum y'^2, sum p'^2, sum pending p^2, non-finite] (one 32-byte NCCL allreduce)
    control update from the global sums               (1-thread kernel, identical on all ranks)

and synchronises once per batch of terms.  That is the NCCL transport.  On one
NVLink / NVSwitch node the default is the peer-memory transport instead: the
fused kernel itself stores its boundary rows of y' into the neighbours'
ghost-row buffers (CUDA IPC mappings) and all-reduces the four term sums through
per-rank boards in peer memory, so a Newton term is ONE kernel launch per rank
with no host call and no collective (``XMHD_STRIP_TRANSPORT=nccl`` selects the
NCCL path).  u's halo rows are exchanged once per phi-call (u is frozen).  Every other norm of the host layer (FD step, error
norm, power iteration, totals) becomes a cross-rank reduction through
``_ops.set_reducer``.

The orchestration (layout, neighbour order, halo ordering, reductions, the
control flow of the Newton loop) is backend-agnostic: ``CudaStripBackend`` runs
the sm_100a kernels; the CPU tests drive the same ``leja_strips`` loop with a
NumPy oracle backend over the gloo transport (tests/test_strips_cpu.py).
"""

import ctypes
import math

import numpy as np
import torch
import torch.distributed as dist

from paper_2108_13622_b200 import _lib
from paper_2108_13622_b200 import _ops

NF = 8
MY, BY = 2, 5


class StripLayout:
    """Balanced contiguous row partition of ny rows over `size` ranks."""

    def __init__(self, ny, size, rank):
        if ny < 2 * size:
            raise ValueError(f"{ny} rows cannot give every one of {size} ranks >= 2 rows")
        base, rem = divmod(ny, size)
        self.counts = [base + (1 if r < rem else 0) for r in range(size)]
        self.starts = [sum(self.counts[:r]) for r in range(size)]
        self.size, self.rank = size, rank
        self.ny_global = ny
        self.y0 = self.starts[rank]
        self.ny = self.counts[rank]

    def local_rows(self, global_fields):
        """(8, ny_global, nx) -> this rank's (8, ny, nx) rows."""
        return global_fields[:, self.y0:self.y0 + self.ny, :]


class Comm:
    """The transport of the decomposition: torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.size = dist.get_world_size(group)
        else:
            self.rank, self.size = 0, 1
        # gloo moves CUDA tensors through collectives but not through send / recv:
        # point-to-point messages of device tensors are staged through the host
        # (the CPU-backend check of the N>1 paths on one GPU; NCCL needs no staging)
        self._host_p2p = (self.size > 1 and dist.get_backend(group) == "gloo")

    def _p2p_buffers(self, tensors):
        """(tensors to post, copy-back list) for point-to-point messages."""
        if not self._host_p2p:
            return list(tensors), []
        staged = [t.detach().to("cpu").contiguous() if t.is_cuda else t for t in tensors]
        return staged, [(t, h) for t, h in zip(tensors, staged) if t.is_cuda]

    def allreduce_sum(self, t):
        if self.size > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def allreduce_max(self, t):
        if self.size > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t

    def neighbours(self, periodic):
        below = self.rank - 1 if self.rank > 0 else (self.size - 1 if periodic else None)
        above = self.rank + 1 if self.rank < self.size - 1 else (0 if periodic else None)
        return below, above

    def gather_host(self, obj):
        """Every rank's host object, in rank order (final-state assembly only)."""
        if self.size == 1:
            return [obj]
        objs = [None] * self.size
        dist.all_gather_object(objs, obj, group=self.group)
        return objs

    def stream_to_root(self, planes, consume, root=0):
        """Plane f of every rank to `root` in global order (f major, ranks in
        order), one (field, rank) band at a time: ``consume(f, r, host_array)``
        runs on `root` only.  Point-to-point, so `root` never holds more than
        one band (a 16384^2 state is 17 GB; a band 268 MB at 8 ranks)."""
        nf = len(planes)
        if self.size == 1:
            for f in range(nf):
                consume(f, 0, _ops.to_host(planes[f]) if torch.is_tensor(planes[f])
                        else np.asarray(planes[f]))
            return
        shapes = self.gather_host([tuple(planes[0].shape)])
        for f in range(nf):
            for r in range(self.size):
                if r == root and self.rank == root:
                    consume(f, r, _ops.to_host(planes[f]))
                elif self.rank == root:
                    buf = torch.empty(shapes[r][0], dtype=planes[f].dtype,
                                      device="cpu" if self._host_p2p else planes[f].device)
                    dist.recv(buf, src=r, group=self.group)
                    consume(f, r, _ops.to_host(buf))
                elif self.rank == r:
                    (msg,), _ = self._p2p_buffers([planes[f].contiguous()])
                    dist.send(msg, dst=root, group=self.group)

    def exchange_rows(self, send_lo, send_hi, recv_lo, recv_hi, periodic):
        """Send my rows 0,1 down and rows ny-2,ny-1 up; receive the neighbours' rows.

        Posting order is fixed (send up, send down, receive from below, receive
        from above) so that with two ranks on a periodic ring the two messages
        between the same pair are matched in order.
        """
        below, above = self.neighbours(periodic)
        if self.size == 1:
            if periodic:
                recv_lo.copy_(send_hi)
                recv_hi.copy_(send_lo)
            return
        (send_lo, send_hi), _ = self._p2p_buffers([send_lo, send_hi])
        (recv_lo, recv_hi), back = self._p2p_buffers([recv_lo, recv_hi])
        ops = []
        if above is not None:
            ops.append(dist.P2POp(dist.isend, send_hi, above, self.group))
        if below is not None:
            ops.append(dist.P2POp(dist.isend, send_lo, below, self.group))
        if below is not None:
            ops.append(dist.P2POp(dist.irecv, recv_lo, below, self.group))
        if above is not None:
            ops.append(dist.P2POp(dist.irecv, recv_hi, above, self.group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for dev, host in back:
            dev.copy_(host)


class Reducer:
    """Cross-rank reductions for the host layer's norms (installed with _ops.set_reducer)."""

    def __init__(self, comm, device):
        self.comm = comm
        self.device = device

    def sum(self, values):
        t = torch.tensor(values, dtype=torch.float64, device=self.device)
        return self.comm.allreduce_sum(t).tolist()

    def max(self, values):
        t = torch.tensor(values, dtype=torch.float64, device=self.device)
        return self.comm.allreduce_max(t).tolist()


def mirror_rows(rows, lo_side):
    """Ghost rows of a reflecting wall from the 2 boundary rows (MY, BY odd).

    rows: (8, 2, nx) boundary rows in grid order.  Returns (8, 2, nx) ghost rows in
    grid order: below the wall [-2, -1] = s*[row 1, row 0]; above it
    [ny, ny+1] = s*[row ny-1, row ny-2].
    """
    ghost = rows.flip(1).clone()
    ghost[MY] *= -1.0
    ghost[BY] *= -1.0
    return ghost


def global_normal_slice(rng, layout, nx):
    """This rank's slice of rng.standard_normal(8*ny*nx) in the global field-major order.

    The reference draws the power-iteration start vector for the whole state
    (linearize.py:113, harness.py:130).  Every rank draws the whole stream
    (split over its host cores by ``_normals.draw``: same values, same final
    generator state as one draw) and keeps its own rows of every field.
    """
    from paper_2108_13622_b200 import _normals
    out = np.empty((NF, layout.ny, nx))
    flat = out.reshape(NF, -1)
    plane = layout.ny_global * nx
    lo_off, hi_off = layout.y0 * nx, (layout.y0 + layout.ny) * nx

    def sink(i0, vals):
        i1 = i0 + vals.size
        for f in range(NF):
            a, b = max(i0, f * plane + lo_off), min(i1, f * plane + hi_off)
            if a < b:
                flat[f, a - f * plane - lo_off:b - f * plane - lo_off] = vals[a - i0:b - i0]

    _normals.draw(rng, NF * plane, np.empty, sink)
    return out.reshape(-1)


def local_normal_slice(rng, layout, nx, comm):
    """This rank's rows of ``rng.standard_normal(8*ny*nx)``, drawing ONLY them.

    The reference draws the power-iteration start vector for the whole state
    from the run RNG (linearize.py:113, harness.py:130); at 16384^2 that is
    2.1 G normals (17 GB).  Here rank r draws just its 8 field segments
    [f*plane + y0*nx, f*plane + y1*nx): each from a copy of the generator
    advanced (PCG64.advance) to a raw position a margin before the segment's
    expected start (NumPy's ziggurat takes one raw output per normal except on
    a rejection, _normals.RHO), over a window long enough to contain the true
    start.  The segments are then aligned in stream order (field-major, ranks
    in order within a field): the 8 values that follow segment s-1 are located
    inside segment s's draw (_normals._locate), which fixes where its exact
    values begin.  That chain costs one tiny all-gather per segment (8 values
    and a start position), not a full draw per rank.  A segment whose window
    misses its start (a > 6-sigma rejection count) is redrawn from the known
    start of the one before.  Every rank's generator ends in the state the
    single global draw leaves it in.  Values are bit-identical to the global
    draw (tests/test_strips_cpu.py)."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_2108_13622_b200 import _normals as nm
    P, me = comm.size, comm.rank
    bg = rng.bit_generator
    if P == 1 or not isinstance(bg, np.random.PCG64):
        return global_normal_slice(rng, layout, nx)
    state0 = bg.state
    plane = layout.ny_global * nx
    segs = [(f, r, f * plane + layout.starts[r] * nx, layout.counts[r] * nx)
            for f in range(NF) for r in range(P)]

    def guess(start):
        if start == 0:
            return 0, 0
        margin = int(6.0 * math.sqrt(start * nm.RHO_VAR)) + 2048
        return max(0, int(start * (1.0 + nm.RHO)) - margin), 2 * margin + 4096

    def draw(k):
        _, _, start, size = segs[k]
        g0, win = guess(start)
        return g0, win, nm._gen_at(state0, g0).standard_normal(size + win + nm.L_MATCH)

    mine = [k for k, sg in enumerate(segs) if sg[1] == me]
    with ThreadPoolExecutor(max_workers=max(1, min(len(mine), nm.host_threads()))) as pool:
        futs = {k: pool.submit(draw, k) for k in mine}
        out = np.empty((NF, layout.ny, nx))
        flat = out.reshape(NF, -1)
        prev = None     # (raw start, normals to skip, size, continuation) of segment k-1
        scratch = np.empty(1 << 16)
        for k, (f, r, start, size) in enumerate(segs):
            info = None
            if r == me:
                g0, win, buf = futs.pop(k).result()
                d = 0 if k == 0 else nm._locate(buf, win, prev[3])
                if d is None:   # redraw from segment k-1's exact start
                    g = nm._gen_at(state0, prev[0])
                    nm._skip(g, prev[1] + prev[2], scratch)
                    g.standard_normal(out=buf[:size + nm.L_MATCH])
                    g0, d = prev[0], prev[1] + prev[2]
                flat[f] = buf[d:d + size]
                info = (g0, d, buf[d + size:d + size + nm.L_MATCH].copy())
            g0, d, cont = comm.gather_host(info)[r]
            prev = (g0, d, size, cont)
    # the generator's state after the whole global draw, from the last segment's start
    st = None
    if segs[-1][1] == me:
        g = nm._gen_at(state0, prev[0])
        nm._skip(g, prev[1] + prev[2], np.empty(1 << 16))
        st = g.bit_generator.state
    st = comm.gather_host(st)[segs[-1][1]]
    st["has_uint32"] = state0["has_uint32"]
    st["uinteger"] = state0["uinteger"]
    bg.state = st
    return out.reshape(-1)


class HaloSet:
    """Send / receive row buffers of one vector, layout [field][2][nx]."""

    def __init__(self, nx, device, dtype=torch.float64):
        z = lambda: torch.empty((NF, 2, nx), dtype=dtype, device=device)
        self.send_lo, self.send_hi, self.lo, self.hi = z(), z(), z(), z()

    def exchange(self, vec3d, comm, periodic):
        """Fill lo/hi with the neighbours' rows of vec3d (8, ny, nx) (or mirrored rows)."""
        self.send_lo.copy_(vec3d[:, :2, :])
        self.send_hi.copy_(vec3d[:, -2:, :])
        below, above = comm.neighbours(periodic)
        if below is None:
            self.lo.copy_(mirror_rows(self.send_lo, True))
        if above is None:
            self.hi.copy_(mirror_rows(self.send_hi, False))
        comm.exchange_rows(self.send_lo, self.send_hi, self.lo, self.hi, periodic)
        return self.lo, self.hi


class StripMhd:
    """Device MHD right-hand side of one y-strip (the strip counterpart of MhdRhs)."""

    def __init__(self, geometry, params, comm=None):
        from paper_2108_13622_b200.mhd import Boundary
        self.comm = comm or Comm()
        self.layout = StripLayout(geometry.ny, self.comm.size, self.comm.rank)
        self.nx, self.ny = geometry.nx, self.layout.ny
        self.ny_global = geometry.ny
        self.dx, self.dy = geometry.dx, geometry.dy
        self.params = params
        self.n = NF * self.nx * self.ny
        self.periodic_y = params.bc_y is Boundary.PERIODIC
        bcx = _lib.BC_PERIODIC if params.bc_x is Boundary.PERIODIC else _lib.BC_REFLECTING
        self.ctx = _lib.Context(self.nx, self.ny, self.dx, self.dy, params.mu, params.eta,
                                params.kappa, params.gamma, params.mu0, bcx, _lib.BC_HALO)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.state_halo = HaloSet(self.nx, dev)
        self.dir_halo = HaloSet(self.nx, dev)
        self._peer = False
        self._peer_off = False   # set when the peer link could not be verified

    def peer_transport(self):
        """True when the Leja loop runs over peer memory (and the link is set up).

        Real ranks of one node (torch.distributed) use it unless
        XMHD_STRIP_TRANSPORT=nccl; host-thread emulations of ranks cannot (their
        kernels would wait on each other on one GPU) and use the NCCL-style path.
        """
        import os
        if self._peer:
            return True
        if (os.environ.get("XMHD_STRIP_TRANSPORT", "peer") != "peer" or self.comm.size < 2
                or not isinstance(self.comm, Comm) or self.comm.size > 8):
            return False
        if self._peer_off:
            return False
        # Every rank takes part in every gather below whatever happened on it, and
        # all ranks read the same gathered lists, so they agree on the outcome: any
        # failure (allocation, IPC mapping, a probe write that did not arrive) on
        # any rank puts the whole job on the NCCL transport instead of hanging it.
        lib = _lib.load()
        handle = (ctypes.c_char * 64)()
        err = None
        try:
            _lib.check(lib.xmhd_p2p_alloc(self.ctx.h, handle), "xmhd_p2p_alloc")
        except (RuntimeError, OSError) as exc:
            err = str(exc)
        got = self.comm.gather_host((err, bytes(handle)))
        errs = [e for e, _ in got if e]
        if not errs:
            try:
                blob = (ctypes.c_char * (64 * len(got))).from_buffer_copy(
                    b"".join(h for _, h in got))
                _lib.check(lib.xmhd_p2p_connect(self.ctx.h, self.comm.rank, self.comm.size, blob,
                                                int(self.periodic_y)), "xmhd_p2p_connect")
                # (probe value, rank) into row `rank` of every rank's board
                _lib.check(lib.xmhd_p2p_probe(self.ctx.h, 1000.0 + self.comm.rank),
                           "xmhd_p2p_probe")
            except (RuntimeError, OSError) as exc:
                err = str(exc)
            errs = [e for e in self.comm.gather_host(err) if e]   # also: every probe has landed
        if not errs:
            board = (ctypes.c_double * 32)()
            try:
                _lib.check(lib.xmhd_p2p_read_board(self.ctx.h, board), "xmhd_p2p_read_board")
                seen = [(board[4 * q], board[4 * q + 1]) for q in range(self.comm.size)]
                if seen != [(1000.0 + q, float(q)) for q in range(self.comm.size)]:
                    err = f"rank {self.comm.rank}: probe writes of its peers did not arrive ({seen})"
            except (RuntimeError, OSError) as exc:
                err = str(exc)
            errs = [e for e in self.comm.gather_host(err) if e]
        if errs:
            self._peer_off = True
            if self.comm.rank == 0:
                import sys
                print(f"[xmhd] peer-memory strip transport unavailable ({errs[0]}); using NCCL",
                      file=sys.stderr, flush=True)
            return False
        self._peer = True
        return True

    def _set_halo(self, u_halo, d_halo=None):
        lib = _lib.load()
        rc = lib.xmhd_set_halo(self.ctx.h, _lib.ptr(u_halo.lo), _lib.ptr(u_halo.hi),
                               _lib.ptr(d_halo.lo) if d_halo else None,
                               _lib.ptr(d_halo.hi) if d_halo else None)
        _lib.check(rc, "xmhd_set_halo")

    def exchange(self, flat, halo):
        return halo.exchange(flat.reshape(NF, self.ny, self.nx), self.comm, self.periodic_y)

    def __call__(self, flat, out=None):
        u = _ops.as_device(flat).reshape(-1)
        if u.numel() != self.n:
            raise ValueError(f"strip state has {u.numel()} entries, needs {self.n}")
        out = torch.empty_like(u) if out is None else out
        self.exchange(u, self.state_halo)
        self._set_halo(self.state_halo)
        from paper_2108_13622_b200.mhd import bad_cells_buffer
        bad = bad_cells_buffer()
        rc = _lib.load().xmhd_rhs(self.ctx.bind_stream(), _lib.ptr(u), _lib.ptr(out), bad)
        _lib.check(rc, "xmhd_rhs (strip)")
        self.raise_if_nonfinite(rc == _lib.NONFINITE, bad, out.device)
        return out

    def raise_if_nonfinite(self, local_bad, bad, device):
        """Every rank raises the same RhsBlowupError when ANY strip's F is
        non-finite (one scalar all-reduce): the message and ``cells`` name the
        first cells of the whole grid in C order with global row indices and
        the global count, as mhd.py:225-231 reports them on one grid."""
        from paper_2108_13622_b200.mhd import _blowup_error, decode_bad_cells
        if self.comm.size > 1:
            t = torch.tensor([1.0 if local_bad else 0.0], dtype=torch.float64, device=device)
            if not self.comm.allreduce_sum(t).item():
                return
        elif not local_bad:
            return
        count, cells = decode_bad_cells(bad, self.layout.y0) if local_bad else (0, [])
        parts = self.comm.gather_host((count, cells))
        total = sum(c for c, _ in parts)
        merged = sorted(cell for _, cl in parts for cell in cl)
        raise _blowup_error(total, merged[:8])

    # -- per-step diagnostics over all strips (harness.py:105-116, 137-138, 209-211, 243)
    def divb_max(self, u):
        self.exchange(u, self.state_halo)
        self._set_halo(self.state_halo)
        out = ctypes.c_double()
        _lib.check(_lib.load().xmhd_divb(self.ctx.bind_stream(), _lib.ptr(u), None,
                                         ctypes.byref(out)), "xmhd_divb (strip)")
        return _ops.global_max([out.value])[0]

    def field_sums(self, u):
        out = (ctypes.c_double * 8)()
        _lib.check(_lib.load().xmhd_field_sums(self.ctx.bind_stream(), _lib.ptr(u), out),
                   "xmhd_field_sums (strip)")
        return _ops.global_sum(list(out))

    def cfl_speeds(self, u):
        out = (ctypes.c_double * 2)()
        _lib.check(_lib.load().xmhd_cfl_speeds(self.ctx.bind_stream(), _lib.ptr(u), out),
                   "xmhd_cfl_speeds (strip)")
        return _ops.global_max(list(out))

    def jvp(self, u, fu, w, eps):
        """(F(u + eps*w) - F(u))/eps on the strip with the caller's (global) eps."""
        self.exchange(u, self.state_halo)
        self.exchange(w, self.dir_halo)
        self._set_halo(self.state_halo, self.dir_halo)
        out = torch.empty_like(w)
        rc = _lib.load().xmhd_jvp_eps(self.ctx.bind_stream(), _lib.ptr(u), _lib.ptr(fu),
                                      _lib.ptr(w), float(eps), _lib.ptr(out), None)
        _lib.check(rc, "xmhd_jvp_eps")
        return out, rc == _lib.NONFINITE


class CudaStripBackend:
    """The per-term device operations of the strip Leja loop (C-ABI calls)."""

    def __init__(self, mhd, lin):
        self.mhd = mhd
        self.lin = lin
        self.lib = _lib.load()
        self.h = mhd.ctx.bind_stream()
        dev = lin.base_state.device
        # [sum y'^2, sum p'^2, sum pending p^2, non-finite] of this rank
        self.sums = torch.zeros(4, dtype=torch.float64, device=dev)

    def start(self, v, dt, q, theta, tol, xi, coeffs):
        mhd = self.mhd
        mhd.exchange(self.lin.base_state, mhd.state_halo)
        mhd._set_halo(mhd.state_halo, mhd.dir_halo)
        rc = self.lib.xmhd_leja_strip_start(
            self.h, _lib.ptr(self.lin.base_state), _lib.ptr(self.lin.base_rhs),
            float(self.lin._base_norm), _lib.ptr(v), float(dt), float(q), float(theta),
            float(tol), _ptr_d(xi), _ptr_d(coeffs), int(coeffs.size), _lib.ptr(self.sums))
        _lib.check(rc, "xmhd_leja_strip_start")
        return self.sums[:1]

    def start_finalize(self, sums):
        _lib.check(self.lib.xmhd_leja_strip_start_finalize(self.h, _lib.ptr(self.sums)),
                   "xmhd_leja_strip_start_finalize")

    def pack(self, mirror_lo, mirror_hi):
        hs = self.mhd.dir_halo
        rc = self.lib.xmhd_leja_strip_pack(self.h, _lib.ptr(hs.send_lo), _lib.ptr(hs.send_hi),
                                           _lib.ptr(hs.lo), _lib.ptr(hs.hi), int(mirror_lo),
                                           int(mirror_hi))
        _lib.check(rc, "xmhd_leja_strip_pack")
        return hs

    def iterate(self):
        _lib.check(self.lib.xmhd_leja_strip_iterate(self.h, _lib.ptr(self.sums)),
                   "xmhd_leja_strip_iterate")
        return self.sums

    def finalize(self, sums):
        _lib.check(self.lib.xmhd_leja_strip_finalize(self.h, _lib.ptr(self.sums)),
                   "xmhd_leja_strip_finalize")

    def state(self):
        st = _lib.LejaState()
        _lib.check(self.lib.xmhd_leja_query(self.h, ctypes.byref(st)), "xmhd_leja_query")
        return st

    def set_coeffs(self, coeffs):
        _lib.check(self.lib.xmhd_leja_set_coeffs(self.h, _ptr_d(coeffs), int(coeffs.size)),
                   "xmhd_leja_set_coeffs")

    def result(self, like):
        p = torch.empty_like(like)
        _lib.check(self.lib.xmhd_leja_result(self.h, _lib.ptr(p)), "xmhd_leja_result")
        return p

    def current_y(self, like):
        y = torch.empty_like(like)
        _lib.check(self.lib.xmhd_leja_current_y(self.h, _lib.ptr(y)), "xmhd_leja_current_y")
        return y


def _ptr_d(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def leja_strips(backend, comm, periodic, l, v, dt, q, theta, tol, xi, coeff_fn, grow_fn,
                batch0=2, batch_max=32):
    """The Newton/Leja loop of leja.py:103-150 on y-strips (backend-agnostic).

    coeff_fn(chunk) -> the initial coefficient array; grow_fn(chunk, coeffs, m)
    -> (chunk, coeffs) on NEED_COEFFS (leja.py:128-130).  Returns the backend's
    final state.  All ranks run the same sequence of collectives.
    """
    below, above = comm.neighbours(periodic)
    chunk = 64
    coeffs = coeff_fn(chunk)
    part = backend.start(v, dt, q, theta, tol, xi, coeffs)
    comm.allreduce_sum(part)
    backend.start_finalize(part)
    batch = batch0
    while True:
        for _ in range(batch):
            hs = backend.pack(below is None, above is None)
            comm.exchange_rows(hs.send_lo, hs.send_hi, hs.lo, hs.hi, periodic)
            sums = backend.iterate()
            comm.allreduce_sum(sums)
            backend.finalize(sums)
        st = backend.state()
        if st.status == _lib.LEJA_NEED_COEFFS:
            chunk, coeffs = grow_fn(chunk, coeffs, st.m)
            backend.set_coeffs(coeffs)
            batch = batch0
            continue
        if st.status != _lib.LEJA_RUNNING:
            return st
        batch = min(2 * batch, batch_max)


def leja_peer(mhd, lin, l, vd, dt, q, theta, tol, xi):
    """The Leja loop over peer memory: one fused launch per term on every rank."""
    from paper_2108_13622_b200 import leja
    lib = _lib.load()
    mhd.exchange(lin.base_state, mhd.state_halo)
    mhd._set_halo(mhd.state_halo, mhd.dir_halo)
    h = mhd.ctx.bind_stream()
    coeffs = np.ascontiguousarray(leja._newton_coeffs(l, q, theta, 64))
    rc = lib.xmhd_leja_p2p_start(h, _lib.ptr(lin.base_state), _lib.ptr(lin.base_rhs),
                                 float(lin._base_norm), _lib.ptr(vd), float(dt), float(q),
                                 float(theta), float(tol), _ptr_d(xi), _ptr_d(coeffs),
                                 int(coeffs.size))
    _lib.check(rc, "xmhd_leja_p2p_start")
    return leja.drive_fused(lib, h, l, q, theta, coeffs, peer=True)


def apply_phi_leja_strips(l, lin, v, dt, shift, tol, xi):
    """apply_phi_leja for a linearization whose RHS is a StripMhd (called by leja.py)."""
    from paper_2108_13622_b200 import leja
    from paper_2108_13622_b200.linearize import RhsBlowupError
    mhd = lin.mhd
    q, theta = shift.q, shift.theta
    vd = _ops.as_device(v).reshape(-1)
    backend = CudaStripBackend(mhd, lin)
    if mhd.peer_transport():
        st = leja_peer(mhd, lin, l, vd, dt, q, theta, tol, xi)
        return _finish(l, lin, mhd, backend, vd, v, st)

    def coeff_fn(chunk):
        c = np.ascontiguousarray(leja._newton_coeffs(l, q, theta, chunk))
        leja._speculate(l, q, theta, min(2 * chunk, leja.LEJA_MAX))
        return c

    grown = []

    def grow_fn(chunk, coeffs, m):
        # the cache insert waits for the call's end (lookahead: term m may
        # never have happened in the reference, leja._grow_pending)
        chunk, table, computed = leja._grow_pending(l, q, theta, chunk, m)
        grown.append((m, table, computed))
        leja._speculate(l, q, theta, min(2 * chunk, leja.LEJA_MAX))
        return chunk, np.ascontiguousarray(table)

    st = leja_strips(backend, mhd.comm, mhd.periodic_y, l, vd, dt, q, theta, tol, xi,
                     coeff_fn, grow_fn)
    leja._commit_growth(l, q, theta, grown, st.iterations)
    leja._drop_speculation(l, q, theta)
    return _finish(l, lin, mhd, backend, vd, v, st)


def _finish(l, lin, mhd, backend, vd, v, st):
    from paper_2108_13622_b200 import leja
    from paper_2108_13622_b200.linearize import RhsBlowupError
    lin.rhs.calls += st.rhs_calls
    if st.status == _lib.LEJA_RHS_NONFINITE:
        y = backend.current_y(vd)
        x = _ops.lincomb((1.0, st.eps), (lin.base_state, y))
        try:
            mhd(x)
        except RhsBlowupError as err:
            raise err
        raise RhsBlowupError("non-finite rhs inside the fused Leja iteration (another strip)")
    p = backend.result(vd)
    return leja.PhiApplyResult(vector=_ops.like(p, v), iterations=int(st.iterations),
                               converged=st.status == _lib.LEJA_CONVERGED,
                               residual=float(st.residual))


def _planes(local_flat, layout, nx):
    if not torch.is_tensor(local_flat):
        local_flat = torch.from_numpy(np.ascontiguousarray(local_flat, dtype=np.float64))
    x = local_flat.reshape(NF, layout.ny * nx)
    return [x[f] for f in range(NF)]


def gather_strips(local_flat, layout, nx, comm, root=0):
    """Full (8, ny, nx) host array on `root` (None elsewhere) from every rank's
    strip, received band by band (Comm.stream_to_root; no pickled state)."""
    full = np.empty((NF, layout.ny_global, nx)) if comm.rank == root else None

    def put(f, r, band):
        y0 = layout.starts[r]
        full[f, y0:y0 + layout.counts[r]] = band.reshape(layout.counts[r], nx)

    comm.stream_to_root(_planes(local_flat, layout, nx), put, root)
    return full


def strip_checksum(local_flat, layout, nx, comm, root=0):
    """sha256 of the GLOBAL flat state (harness.py:118-119: little-endian f8 in
    field-major order) fed band by band on `root` ("" elsewhere): the checksum
    of a 17 GB state without assembling it anywhere."""
    import hashlib
    h = hashlib.sha256() if comm.rank == root else None

    def put(f, r, band):
        h.update(np.ascontiguousarray(band, dtype="<f8").tobytes())

    comm.stream_to_root(_planes(local_flat, layout, nx), put, root)
    return h.hexdigest() if h is not None else ""


def strip_norm_check(x_local, comm):
    """||x|| of a distributed vector (diagnostics helper)."""
    s = _ops.sumsq(x_local)
    return math.sqrt(comm.allreduce_sum(torch.tensor([s], dtype=torch.float64,
                                                     device=x_local.device)).item())
