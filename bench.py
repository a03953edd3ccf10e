"""Benchmark of the B200 Leja phi-action hot path (BASELINE.json configs[1]).

Workload (one "step"): phi_1(dt J(u)) v on the 2048^2 config-1 state (KH +
seeded Fourier modes, fp64, 8 fields), v a seeded unit Gaussian, swept over
alpha*dt in {1, 10, 100, 300} (Leja degree ~10-240), Leja tol 1e-10, the
coefficient cache cleared per step so the host coefficient work is included.

  value : cell-updates/s = sum(Leja iterations) * nx*ny / device time, inputs
          resident in HBM (state vectors 268 MB each >> 126 MB L2: no flush).
  e2e   : same metric through the public API the reference's callers use:
          plain (pageable) NumPy arrays in, NumPy arrays out; per step u and
          the 4 right-hand vectors go H2D and the 4 results D2H.  ``e2e_pinned``
          is the same with page-locked torch host tensors.
  roofline : the fused Leja iteration kernel: CUDA events on its stream around
          every batch of term launches inside the timed region, divided by the
          Newton terms (``kernel_ms``; ``kernel_ms_alone`` / ``by_kind`` come
          from a burst of back-to-back terms afterwards).  Algorithmic bytes per cell per Newton term:
          320 (lookahead interpolant schedule: an odd term reads u, y, F(u)
          and writes y' = 256 B, the even term reads u, y, F(u), p and writes
          y', p' = 384 B), 384 with XMHD_PDEFER=0; ``by_kind`` gives each term
          kind against its own bytes.
  stencil_kernels : the RHS (128 B/cell) and FD-JVP (256 B/cell) stencil
          kernels of the metric's "RHS/Jv", timed the same way (N=1 only).
  scale_case : north_star's strong-scaling case: phi_1(dt J) F(u)/||F(u)|| on
          the 8192^2 Harris state of config 4 (alpha*dt in {1, 10, 100}),
          y-strips over the N ranks, each rank building only its own rows.
  cpu_baseline : the NumPy oracle (the reference's own algorithm, oracle/) on a
          bounded sample of the same workload on this host.

``--gpus N`` without a torchrun environment re-launches itself under
``torch.distributed.run`` (N ranks, 127.0.0.1), after checking that N GPUs are
visible (it fails loudly otherwise instead of timing one GPU).  Under N>1 the
2048^2 grid is split into y-strips (2-row halo + one 4-scalar all-reduce per
Leja term inside the fused kernel over peer memory, or NCCL,
paper_2108_13622_b200/strips.py); the total work is fixed ("scaling":
"strong") and `value` is whole-job cell-updates/s over the max-over-ranks
device time.  ``--impl reference`` times that CPU implementation alone (rank
0; other ranks exit 0).
"""

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "RHS/Jv cell-updates/s (fp64 GB/s vs HBM peak); wall-s per EXPRB step"
SWEEP = (1.0, 10.0, 100.0, 300.0)
LEJA_TOL = 1e-10
# XMHD_BENCH_SHARED_GPU=1: N ranks share device 0 over gloo (a check of the N>1
# host logic where only one GPU exists; its line says so and is not a measurement)
SHARED_GPU = bool(int(os.environ.get("XMHD_BENCH_SHARED_GPU", "0") or "0"))
# algorithmic bytes per cell per Newton term
def bytes_per_cell_term(world):
    return 384.0 if os.environ.get("XMHD_PDEFER", "1") == "0" else 320.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", "--grid", dest="n", type=int, default=2048,
                    help="grid size (config 1: 2048)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-exprb", action="store_true")
    ap.add_argument("--no-scale-case", action="store_true")
    ap.add_argument("--scale-n", type=int, default=8192, help="scale_case grid (config 4: 8192)")
    return ap.parse_args()


def maybe_spawn(args):
    """--gpus N > 1 outside torchrun: re-launch under torch.distributed.run, or
    fail loudly when fewer than N GPUs are visible (never time N=1 silently).
    Returns an exit code, or None when this process is already a rank."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    if args.impl != "reference" and not SHARED_GPU:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.stderr.write(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) "
                             f"visible; refusing to report a {args.gpus}-GPU number\n")
            return 2
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)]
    # torchrun's own parser would read a bare `--n` as an abbreviation of its options
    for a in sys.argv[1:]:
        cmd.append("--grid" + a[3:] if a == "--n" or a.startswith("--n=") else a)
    return subprocess.call(cmd)


def ncu_traffic(n, local_cells):
    """DRAM bytes per launch of the fused kernel from the committed ncu capture
    (profiles/r02_leja_traffic.json), when it was taken on this grid and layout."""
    path = os.path.join(REPO, "profiles", "r02_leja_traffic.json")
    try:
        rec = json.load(open(path))
    except (OSError, ValueError):
        return None
    if rec.get("grid") != n or local_cells != n * n:
        return None
    return {"bytes": rec["dram_bytes_read"] + rec["dram_bytes_write"],
            "algorithmic_bytes": rec["algorithmic_bytes"], "source": rec["source"]}


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled every 100 ms during the timed region.

    In-process NVML (nvidia_ml_py) from a background thread: a few light
    queries per sample.  A polling nvidia-smi process (the fallback) was seen
    to stall the host-driven launch loop on some boxes (the timed region ran
    1.2-2.3x slower than the same loop unsampled)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.nvml = None
        self.lines = []
        self._stop = threading.Event()

    def _nvml_handle(self, nv):
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            return nv.nvmlDeviceGetHandleByPciBusId_v2(bus)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def _nvml_sample(self):
        nv, h = self.nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        flags = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                 nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        act = ["Active" if r & f else "Not Active" for f in flags]
        return ", ".join([str(sm), str(smax), "0"] + act)

    def _nvml_loop(self):
        while not self._stop.wait(0.1):
            try:
                self.lines.append(self._nvml_sample())
            except Exception:
                return

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nvml = (nv, self._nvml_handle(nv))
            self._nvml_sample()   # first query outside the timed region
            self.thread = threading.Thread(target=self._nvml_loop, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # let nvidia-smi finish starting up (process spawn, NVML init) before
            # the timed region begins, so it does not compete with the host side
            t0 = time.perf_counter()
            while len(self.lines) < 2 and time.perf_counter() - t0 < 20.0:
                time.sleep(0.01)
            self.lines.clear()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.nvml is not None:
            self._stop.set()
            self.thread.join(timeout=2)
            try:
                self.lines.append(self._nvml_sample())   # the region's last state
            except Exception:
                pass
            return
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = max(smax, float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": smax or None, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_sample(n, iters=3, adt=10.0):
    """The NumPy oracle (reference algorithm) on `iters` Leja iterations of the workload.

    Threading as the reference gets it: NumPy's elementwise ufuncs (nearly all
    of the work) run on one core; OpenBLAS's ddot (the norms) may use every
    core of the host (not limited here)."""
    threads = os.cpu_count() or 1
    try:
        from threadpoolctl import threadpool_info
        threads = max([threads] + [int(i.get("num_threads", 1)) for i in threadpool_info()])
    except Exception:
        pass
    from oracle import leja_np as olj, mhd_np
    from paper_2108_13622_b200 import scenarios as sc
    s = sc.CONFIGS[1]()
    s.nx = s.ny = n
    q = sc.initial_fields(s)

    def f(flat):
        return mhd_np.rhs(flat.reshape(q.shape), s.dx, s.dy, s.mu, s.eta, s.kappa)
    lin = olj.Frozen(olj.CountedRhs(f), q.reshape(-1))
    v = sc.unit_gaussian(q.size, s.extra["v_seed"])
    alpha = 5855.0 * (n / 2048.0) ** 2   # survey-measured alpha scale; only sets q, theta
    dt = adt / alpha
    qq, th = olj.shift_scale(alpha * dt)
    xi = olj.leja_points(500)
    c = olj.CoeffCache().get(1, qq, th, 64)
    y = v.copy()
    p = c[0] * y
    t0 = time.perf_counter()
    for m in range(1, iters + 1):
        w = olj.fd_jvp(lin, y)
        y = (dt * w - qq * y) / th - xi[m - 1] * y
        ny = np.linalg.norm(y)
        p = p + c[m] * y
        _ = abs(c[m]) * ny / max(1.0, np.linalg.norm(p))
    wall = time.perf_counter() - t0
    model = ""
    try:
        with open("/proc/cpuinfo") as fh:
            model = next((l.split(":", 1)[1].strip() for l in fh if l.startswith("model name")), "")
    except OSError:
        pass
    return {"value": iters * n * n / wall, "unit": "cell-updates/s", "cores": threads,
            "kind": "port", "cpu_model": model, "host_cpus": os.cpu_count(),
            "sample": f"{iters} Leja iterations (FD-JVP + Newton update + 2 norms) of the "
                      f"config-1 phi_1 call at {n}^2, alpha*dt={adt:g}, NumPy oracle (the "
                      f"reference's algorithm and ufunc sequence): ufuncs on 1 core, BLAS "
                      f"norms on up to {threads} threads, {wall:.1f} s"}


def workload_name(n):
    return f"config1: phi_1(dt J)v at {n}^2, alpha*dt sweep {list(SWEEP)}, Leja tol {LEJA_TOL:g}"


def workload_config(n):
    """The `config` dict of BOTH arms (same workload, same keys)."""
    return {"workload": workload_name(n), "grid": n, "alpha_dt": list(SWEEP),
            "leja_tol": LEJA_TOL, "l2_policy": "inputs larger than L2 (268 MB per vector)"}


DATA = ("synthetic (seeded BASELINE config-1 state: KH 2048^2 + 16 Fourier modes per field; "
        "v seeded unit Gaussian)")


def reference_arm(args, rank, world):
    if rank != 0:
        return
    try:
        # torchrun exports OMP_NUM_THREADS=1 to its ranks: give the BLAS norms
        # of the reference path every core again
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=os.cpu_count() or 1)
    except Exception:
        pass
    iters = max(1, args.steps)
    t0 = time.perf_counter()
    samples = []
    for k in range(args.warmup + iters):
        r = cpu_sample(args.n, iters=1)
        if k >= args.warmup:
            samples.append(r["value"])
    value = float(np.mean(samples))
    cores = r["cores"]
    wall = time.perf_counter() - t0
    line = {"metric": METRIC, "value": value, "unit": "cell-updates/s", "n_gpus": world,
            "steps": iters, "warmup": args.warmup, "ms_per_step": 1e3 * args.n ** 2 / value,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": DATA, "impl": "reference",
            "config": workload_config(args.n),
            "parallelism": "cpu (reference NumPy path: ufuncs on one core, BLAS norms "
                           "multi-threaded); rank 0 only",
            "sampling": "each step = 1 Leja term (FD-JVP + Newton update + 2 norms) of the "
                        "alpha*dt=10 call; the metric is per cell-update, so the sweep's rate "
                        "is the per-term rate",
            "cpu_baseline": {"value": value, "unit": "cell-updates/s", "cores": cores,
                             "kind": "port",
                             "sample": f"1 Leja iteration per step at {args.n}^2 via the NumPy "
                                       f"oracle (ufuncs on one core, BLAS norms on up to "
                                       f"{cores} threads), total {wall:.1f} s"},
            "e2e": {"value": value, "unit": "cell-updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def total_launches(op=None):
    from paper_2108_13622_b200 import _ops, mhd
    ctxs = list(mhd._ctx_cache.values()) + list(_ops._util.values())
    if op is not None and op.ctx not in ctxs:
        ctxs.append(op.ctx)
    return sum(c.launches() for c in ctxs)


class Job:
    """Rank / device plumbing shared by the bench parts."""

    def __init__(self, world, rank, local):
        import torch
        import torch.distributed as dist
        self.world, self.rank, self.local = world, rank, local
        self.torch, self.dist = torch, dist
        self.comm = None

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def maxed(self, x):
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def domain(self, xb, setup, params):
        """(RHS operator, this rank's initial rows on the device) of a Setup."""
        from paper_2108_13622_b200 import scenarios as sc, strips
        if self.world > 1:
            if self.comm is None:
                self.comm = strips.Comm()
                xb.linearize._ops.set_reducer(
                    strips.Reducer(self.comm, self.torch.device("cuda", self.local)))
            mhd = strips.StripMhd(xb.StateGrid(setup.nx, setup.ny, setup.dx, setup.dy, None),
                                  params, self.comm)
            rows = (mhd.layout.y0, mhd.layout.y0 + mhd.layout.ny)
            q = sc.initial_fields(setup, rows)
            u = self.torch.from_numpy(q).cuda().reshape(-1)
            return mhd, u, rows
        q = sc.initial_fields(setup)
        u = self.torch.from_numpy(q).cuda().reshape(-1)
        st = xb.StateGrid(setup.nx, setup.ny, setup.dx, setup.dy, u.reshape(8, setup.ny, setup.nx))
        return xb.MhdRhs(st, params), u, None

    def transport(self, mhd):
        if self.world == 1:
            return "single-gpu"
        kind = "peer memory (CUDA IPC)" if mhd.peer_transport() else "NCCL"
        return f"y-strips x{self.world} ({kind}: 2-row halo + 4-scalar all-reduce per term)"


def main():
    args = parse()
    world, rank, local = dist_setup()
    rc = maybe_spawn(args) if world == 1 else None
    if rc is not None:
        sys.exit(rc)
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    if SHARED_GPU and world > 1:
        # host-logic check of the N>1 paths on a one-GPU box: every rank on device
        # 0, gloo, the torch.distributed strip transport (no kernel waits on a peer)
        local = 0
        os.environ["XMHD_STRIP_TRANSPORT"] = "nccl"
    torch.cuda.set_device(local)
    if world > 1:
        if SHARED_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    job = Job(world, rank, local)

    import paper_2108_13622_b200 as xb
    from paper_2108_13622_b200 import _lib, leja, scenarios as sc

    s = sc.CONFIGS[1]()
    s.nx = s.ny = args.n
    n_cells = s.nx * s.ny
    params = xb.MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa)
    mhd, u_dev, rows = job.domain(xb, s, params)
    v_full = sc.unit_gaussian(8 * n_cells, s.extra["v_seed"]).reshape(8, s.ny, s.nx)
    v_loc = np.ascontiguousarray(v_full if rows is None else v_full[:, rows[0]:rows[1]])
    del v_full
    v_dev = torch.from_numpy(v_loc).cuda().reshape(-1)
    op = xb.RhsOperator(mhd)
    lin = xb.FrozenLinearization(op, u_dev)
    est = xb.estimate_alpha(lin, None, rng=np.random.default_rng(0))
    alpha = est.alpha
    matvec = xb.JacobianAction(lin)

    def sweep(vec):
        its = 0
        outs = []
        for adt in SWEEP:
            dt = adt / alpha
            res = xb.apply_phi_leja(1, matvec, vec, dt, xb.shift_and_scale(alpha * dt), LEJA_TOL)
            its += res.iterations
            outs.append(res)
        return its, outs

    # ---- device-resident timed region
    for _ in range(args.warmup):
        leja._coeff_cache.clear()
        sweep(v_dev)
    stream = torch.cuda.current_stream()
    iters_total = 0
    degrees = None
    launches0 = total_launches(mhd)
    # the fused terms' device time inside the timed region: CUDA events on the
    # library's stream around every batch of term launches (xmhd_term_timing)
    _lib.check(_lib.load().xmhd_term_timing(mhd.ctx.bind_stream(), 1, None), "xmhd_term_timing")
    with ClockSampler(local) as clocks:
        job.barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            leja._coeff_cache.clear()
            its, outs = sweep(v_dev)
            iters_total += its
            degrees = [r.iterations for r in outs]
        ev1.record(stream)
        job.barrier()
    launches = total_launches(mhd) - launches0
    ms = job.maxed(ev0.elapsed_time(ev1))
    term_ms = ctypes.c_double()
    _lib.check(_lib.load().xmhd_term_timing(mhd.ctx.bind_stream(), 0, ctypes.byref(term_ms)),
               "xmhd_term_timing")
    term_ms = job.maxed(term_ms.value)
    # every rank processes its strip of the same iterations: whole-job cell-updates
    value = iters_total * n_cells / (ms * 1e-3)

    # ---- the dominant kernel alone: CUDA events around back-to-back fused iterations
    # (single domain only: a strip's terms need its neighbours' ghost rows and sums)
    alone_ms, kind_ms = (time_fused_iteration(xb, _lib, lin, mhd, v_dev, alpha) if world == 1
                         else (None, None))
    # roofline: the average term inside the timed region; the torch.distributed
    # strip loop is not bracketed, there the whole region / terms is the upper bound
    kern_ms = term_ms / iters_total if term_ms > 0.0 else ms / iters_total
    # single domain only: in y-strip mode the stencil needs exchanged ghost rows
    stencil_ms = time_stencil_modes(_lib, lin, mhd, v_dev) if world == 1 else {}
    local_cells = u_dev.numel() // 8
    bpc = bytes_per_cell_term(world)
    achieved = bpc * local_cells / (kern_ms * 1e-3) / 1e9
    peak, peak_kind = measured_peaks()

    # ---- end to end through the public API: NumPy in, NumPy out (pageable,
    # as the reference's callers hold their arrays), and page-locked tensors
    q_loc = np.ascontiguousarray(u_dev.reshape(8, -1, s.nx).cpu().numpy())

    def e2e_step(u_host, v_host):
        its = 0
        leja._coeff_cache.clear()
        op_e = xb.RhsOperator(mhd)
        lin_e = xb.FrozenLinearization(op_e, u_host)            # H2D u, F(u)
        for adt in SWEEP:
            dt = adt / alpha
            res = xb.apply_phi_leja(1, xb.JacobianAction(lin_e), v_host, dt,
                                    xb.shift_and_scale(alpha * dt), LEJA_TOL)   # H2D v, D2H p
            assert isinstance(res.vector, np.ndarray)
            its += res.iterations
        return its

    def e2e_timed(u_host, v_host):
        for _ in range(args.warmup):
            e2e_step(u_host, v_host)
        e2e_iters = 0
        job.barrier()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_iters += e2e_step(u_host, v_host)
        e1.record(stream)
        job.barrier()
        e_ms = job.maxed(max(e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t0)))
        vec_bytes = 8 * 8 * n_cells   # whole job: every rank moves its strip
        return {"value": e2e_iters * n_cells / (e_ms * 1e-3), "unit": "cell-updates/s",
                "h2d_bytes_per_step": vec_bytes * (1 + len(SWEEP)),
                "d2h_bytes_per_step": vec_bytes * len(SWEEP), "ms_per_step": e_ms / args.steps}

    e2e = e2e_timed(q_loc.reshape(-1), v_loc.reshape(-1))
    e2e["inputs"] = "pageable NumPy arrays (the reference callers' containers)"
    e2e_pinned = e2e_timed(torch.from_numpy(q_loc.reshape(-1)).pin_memory(),
                           torch.from_numpy(v_loc.reshape(-1)).pin_memory())
    e2e_pinned["inputs"] = "page-locked torch host tensors"
    del q_loc

    scale = None
    if not args.no_scale_case:
        scale = scale_case(xb, job, args, peak)

    exprb = exprb_c2 = None
    if not args.no_exprb and rank == 0 and world == 1:
        exprb = exprb_step_time(xb, with_cpu=not args.no_cpu_baseline)
        exprb_c2 = exprb_step_time_c2(xb, with_cpu=not args.no_cpu_baseline)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_sample(args.n)

    if rank == 0:
        plan = mhd.ctx.plan()
        kinds = None
        if kind_ms is not None:
            kinds = {k: {"kernel_ms": t, "bytes_per_cell": b,
                         "achieved": b * local_cells / (t * 1e-3) / 1e9,
                         "frac": b * local_cells / (t * 1e-3) / 1e9 / peak}
                     for k, t, b in (("odd_PM_SKIP", kind_ms[0], 256.0),
                                     ("even_PM_LOOK", kind_ms[1], 384.0))}
        line = {
            "metric": METRIC, "value": value, "unit": "cell-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": DATA,
            "config": workload_config(args.n),
            "parallelism": job.transport(mhd),
            "workload_detail": {"alpha": alpha, "leja_degrees": degrees, "stencil_plan": plan},
            "gbs_algorithmic": value * bpc / 1e9,
            "jv_per_s": value / n_cells,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_source": peak_kind,
                         # the same term at the reference's 384 B/cell traffic
                         "frac_at_384B": 384.0 * local_cells / (kern_ms * 1e-3) / 1e9 / peak,
                         "kernel": "stencil_kernel<MODE_LEJA> (fused FD-JVP + Newton update)",
                         "kernel_ms": kern_ms, "bytes_per_cell": bpc,
                         "timed": ("CUDA events around every batch of term launches inside the "
                                   "timed region, / Newton terms" if term_ms > 0.0 else
                                   "timed region / Newton terms (upper bound: halo exchange and "
                                   "all-reduce of the torch.distributed transport included)"),
                         "share_of_step": term_ms / ms if term_ms > 0.0 else None,
                         # the same kernel in a burst of 48 back-to-back launches after the
                         # timed region (clocks recover between phases: box- and state-dependent)
                         "kernel_ms_alone": alone_ms,
                         "frac_alone": (bpc * local_cells / (alone_ms * 1e-3) / 1e9 / peak
                                        if alone_ms else None),
                         "by_kind": kinds,
                         "traffic": ncu_traffic(args.n, local_cells)},
            # the other two stencil kernels of the metric's "RHS/Jv", timed the same
            # way (not in the timed step: the phi sweep runs only the fused term)
            "stencil_kernels": {
                k: {"kernel_ms": t, "bytes_per_cell": b,
                    "achieved_gbs": b * local_cells / (t * 1e-3) / 1e9,
                    "frac": b * local_cells / (t * 1e-3) / 1e9 / peak,
                    "cell_updates_per_s": local_cells / (t * 1e-3)}
                for k, (t, b) in stencil_ms.items()},
            "e2e": e2e,
            "e2e_pinned": e2e_pinned,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        if SHARED_GPU and world > 1:
            line["dry_run"] = (f"{world} ranks sharing one GPU over gloo (XMHD_BENCH_SHARED_GPU): "
                               "a check of the N>1 host logic, not a measurement")
        if scale is not None:
            line["scale_case"] = scale
        if exprb is not None:
            line["exprb_step"] = exprb
        if exprb_c2 is not None:
            line["exprb_step_c2"] = exprb_c2
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


SCALE_SWEEP = (1.0, 10.0, 100.0)


def scale_case(xb, job, args, peak):
    """north_star's strong-scaling case at every N: phi_1(dt J(u)) F(u)/||F(u)||
    on config 4's 8192^2 Harris state (eta 1e-3), alpha*dt in {1, 10, 100}, tol
    1e-10; y-strips over the ranks, each building only its rows and drawing only
    its rows of the power-iteration start vector."""
    import torch
    from paper_2108_13622_b200 import _ops, harness, leja, scenarios as sc
    s = sc.CONFIGS[4]()
    s.nx = s.ny = args.scale_n
    n_cells = s.nx * s.ny
    params = xb.MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa)
    t_setup = time.perf_counter()
    mhd, u, rows = job.domain(xb, s, params)
    op = xb.RhsOperator(mhd)
    lin = xb.FrozenLinearization(op, u)
    if job.world == 1:
        rng = harness._PrefetchedNormals(0, u.numel())   # parallel exact draw
    else:
        rng = np.random.default_rng(0)                   # strips: local_normal_slice
    est = xb.estimate_alpha(lin, None, rng=rng)
    alpha = est.alpha
    fn = _ops.norm(lin.base_rhs)
    v = _ops.divide(lin.base_rhs, fn)
    setup_s = time.perf_counter() - t_setup
    matvec = xb.JacobianAction(lin)

    def sweep():
        its, degs = 0, []
        leja._coeff_cache.clear()
        for adt in SCALE_SWEEP:
            dt = adt / alpha
            res = xb.apply_phi_leja(1, matvec, v, dt, xb.shift_and_scale(alpha * dt), LEJA_TOL)
            its += res.iterations
            degs.append(res.iterations)
        return its, degs

    sweep()
    steps = max(1, min(args.steps, 3))
    stream = torch.cuda.current_stream()
    job.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    its = 0
    for _ in range(steps):
        k, degs = sweep()
        its += k
    e1.record(stream)
    job.barrier()
    ms = job.maxed(e0.elapsed_time(e1))
    value = its * n_cells / (ms * 1e-3)
    bpc = bytes_per_cell_term(job.world)
    per_gpu_bytes = bpc * (its * n_cells / job.world)
    out = {"workload": f"config4 state: Harris {s.nx}^2 eta 1e-3; phi_1(dt J)F(u)/||F(u)||, "
                       f"alpha*dt {list(SCALE_SWEEP)}, Leja tol {LEJA_TOL:g}",
           "grid": s.nx, "n_gpus": job.world, "scaling": "strong",
           "parallelism": job.transport(mhd), "value": value, "unit": "cell-updates/s",
           "ms_per_step": ms / steps, "steps": steps, "leja_degrees": degs, "alpha": alpha,
           "gbs_per_gpu_algorithmic": per_gpu_bytes / (ms * 1e-3) / 1e9,
           "frac_per_gpu": per_gpu_bytes / (ms * 1e-3) / 1e9 / peak,
           "setup_s": setup_s,
           "setup": "each rank builds only its rows of the initial state and of the "
                    "power-iteration start vector (scenarios.initial_fields(rows), "
                    "strips.local_normal_slice)" if job.world > 1 else
                    "whole grid on one GPU; start vector drawn on host threads"}
    del lin, op, u, v, est
    torch.cuda.empty_cache()
    return out


def time_stencil_modes(_lib, lin, mhd, v_dev, n_iter=40):
    """Average duration (CUDA events on the context stream) of the RHS stencil
    (F(u), 128 B/cell: read u, write F) and of the FD-JVP stencil (256 B/cell:
    read u, w, F(u), write Jw), each launched back to back (xmhd_time_stencil)."""
    import ctypes
    import torch
    lib = _lib.load()
    out = torch.empty_like(v_dev)
    res = {}
    for name, mode, b in (("rhs", 0, 128.0), ("jvp", 1, 256.0)):
        ms = ctypes.c_double()
        rc = lib.xmhd_time_stencil(mhd.ctx.bind_stream(), mode, _lib.ptr(lin.base_state),
                                   _lib.ptr(lin.base_rhs), float(lin._base_norm),
                                   _lib.ptr(v_dev), _lib.ptr(out), int(n_iter), ctypes.byref(ms))
        _lib.check(rc, "xmhd_time_stencil")
        res[name] = (float(ms.value), b)
    torch.cuda.synchronize()
    return res


def time_fused_iteration(xb, _lib, lin, mhd, v_dev, alpha, n_iter=48):
    """Average duration of the fused Leja iteration kernel (CUDA events, same
    stream), and the per-kind averages (odd PM_SKIP, even PM_LOOK terms) from
    a second run with an event between launches."""
    import ctypes
    import torch
    from paper_2108_13622_b200 import leja
    adt = 10.0
    dt = adt / alpha
    sh = xb.shift_and_scale(alpha * dt)
    coeffs = np.ascontiguousarray(leja._newton_coeffs(1, sh.q, sh.theta, 500))
    xi = np.ascontiguousarray(leja.leja_points(500))
    out = ctypes.c_double()
    lib = _lib.load()
    dp = ctypes.POINTER(ctypes.c_double)
    rc = lib.xmhd_time_leja_iterations(mhd.ctx.bind_stream(), _lib.ptr(lin.base_state),
                                       _lib.ptr(lin.base_rhs), float(lin._base_norm),
                                       _lib.ptr(v_dev), float(dt), float(sh.q), float(sh.theta),
                                       xi.ctypes.data_as(dp), coeffs.ctypes.data_as(dp),
                                       int(n_iter), ctypes.byref(out), None)
    _lib.check(rc, "xmhd_time_leja_iterations")
    kinds = (ctypes.c_double * 2)()
    per = ctypes.c_double()
    rc = lib.xmhd_time_leja_iterations(mhd.ctx.bind_stream(), _lib.ptr(lin.base_state),
                                       _lib.ptr(lin.base_rhs), float(lin._base_norm),
                                       _lib.ptr(v_dev), float(dt), float(sh.q), float(sh.theta),
                                       xi.ctypes.data_as(dp), coeffs.ctypes.data_as(dp),
                                       int(n_iter), ctypes.byref(per), kinds)
    _lib.check(rc, "xmhd_time_leja_iterations")
    torch.cuda.synchronize()
    return float(out.value), (float(kinds[0]), float(kinds[1]))


def exprb_step_time(xb, with_cpu=False):
    """Config 0 (KH 128^2, EXPRB43, tol 1e-4, t_end 0.5): wall-s per accepted step."""
    from paper_2108_13622_b200 import leja, scenarios as sc
    import torch
    setup = sc.kh_setup(128)
    xb.run(xb.RunConfig(scenario=sc.kh_setup(128, t_final=0.02), tol=setup.tol))  # warm
    leja._coeff_cache.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = xb.run(xb.RunConfig(scenario=setup, scheme=xb.Scheme.EXPRB43, tol=setup.tol))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    out = {"config": "config0 KH 128^2 EXPRB43 tol 1e-4 t_end 0.5",
           "accepted": rep.accepted, "rejected": rep.rejected, "rhs_evals": rep.rhs_evals,
           "wall_s": wall, "wall_s_per_step": wall / max(rep.accepted, 1)}
    if with_cpu:
        out["cpu_baseline"] = exprb_cpu_time(setup)
    return out


def exprb_step_time_c2(xb, with_cpu=False):
    """Config 2 (double Harris 512^2, EXPRB54s4, tol 1e-6, t_end 10): wall-s
    per accepted step over the whole run; the CPU side is the oracle's first
    step (a bounded sample: the whole reference run takes ~47 min)."""
    from paper_2108_13622_b200 import leja, scenarios as sc
    import torch
    setup = sc.CONFIGS[2]()
    xb.run(xb.RunConfig(scenario=sc.harris_setup(512, t_final=0.05), scheme=xb.Scheme.EXPRB54S4,
                        tol=setup.tol))   # warm
    leja._coeff_cache.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = xb.run(xb.RunConfig(scenario=setup, scheme=xb.Scheme.EXPRB54S4, tol=setup.tol))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    out = {"config": "config2 Harris 512^2 EXPRB54s4 tol 1e-6 t_end 10",
           "accepted": rep.accepted, "rejected": rep.rejected, "rhs_evals": rep.rhs_evals,
           "wall_s": wall, "wall_s_per_step": wall / max(rep.accepted, 1)}
    if with_cpu:
        from oracle import steppers_np as ost
        q = sc.initial_fields(setup)
        t0 = time.perf_counter()
        crep = ost.run(q, setup.dx, setup.dy, setup.mu, setup.eta, setup.kappa, "exprb54s4",
                       setup.tol, setup.t_final, max_accepted=1)
        cw = time.perf_counter() - t0
        out["cpu_baseline"] = {"kind": "port", "accepted": crep.accepted,
                               "rhs_evals": crep.rhs_evals, "wall_s": cw,
                               "wall_s_per_step": cw / max(crep.accepted, 1),
                               "sample": "the first step of the same run (incl. its spectral "
                                         "estimate) through the NumPy oracle"}
    return out


def exprb_cpu_time(setup):
    """The same adaptive run through the NumPy oracle (the reference's algorithm
    and ufunc sequence) on this host: wall-s per accepted step, beside ours."""
    from oracle import steppers_np as ost
    from paper_2108_13622_b200 import scenarios as sc
    q = sc.initial_fields(setup)
    t0 = time.perf_counter()
    rep = ost.run(q, setup.dx, setup.dy, setup.mu, setup.eta, setup.kappa, "exprb43", setup.tol,
                  setup.t_final)
    wall = time.perf_counter() - t0
    return {"kind": "port", "accepted": rep.accepted, "rhs_evals": rep.rhs_evals,
            "wall_s": wall, "wall_s_per_step": wall / max(rep.accepted, 1),
            "sample": "the whole config-0 run (same step sequence) through the NumPy oracle"}


if __name__ == "__main__":
    main()
