"""Benchmark of the B200 Leja phi-action hot path (BASELINE.json configs[1]).

Workload (one "step"): phi_1(dt J(u)) v on the 2048^2 config-1 state (KH +
seeded Fourier modes, fp64, 8 fields), v a seeded unit Gaussian, swept over
alpha*dt in {1, 10, 100, 300} (Leja degree ~10-240), Leja tol 1e-10, the
coefficient cache cleared per step so the host coefficient work is included.

  value : cell-updates/s = sum(Leja iterations) * nx*ny / device time, inputs
          resident in HBM (state vectors 268 MB each >> 126 MB L2: no flush).
  e2e   : same metric through the public API with pinned HOST buffers: per step
          u and the 4 right-hand vectors are copied H2D and the 4 results D2H.
  roofline : the fused Leja iteration kernel, timed with CUDA events on its
          stream.  Algorithmic bytes per cell per Newton term:
          320 (lookahead interpolant schedule: an odd term reads u, y, F(u)
          and writes y' = 256 B, the even term reads u, y, F(u), p and writes
          y', p' = 384 B), 384 with XMHD_PDEFER=0.
  stencil_kernels : the RHS (128 B/cell) and FD-JVP (256 B/cell) stencil
          kernels of the metric's "RHS/Jv", timed the same way (N=1 only).
  cpu_baseline : the NumPy oracle (the reference's own algorithm, oracle/) on a
          bounded sample of the same workload on this host.

``--impl reference`` times that CPU implementation alone (rank 0; other ranks
exit 0).  N>1 under torchrun: one process per GPU, the 2048^2 grid split into
y-strips (2-row NCCL halo exchange + one 3-scalar allreduce per Leja term,
paper_2108_13622_b200/strips.py); the total work is fixed ("scaling": "strong")
and `value` is whole-job cell-updates/s over the max-over-ranks device time.
"""

import argparse
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
# algorithmic bytes per cell per Newton term
def bytes_per_cell_term(world):
    return 384.0 if os.environ.get("XMHD_PDEFER", "1") == "0" else 320.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=2048, help="grid size (config 1: 2048)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-exprb", action="store_true")
    return ap.parse_args()


def ncu_traffic(n, local_cells):
    """DRAM bytes per launch of the fused kernel from the committed ncu capture
    (profiles/r01_leja_traffic.json), when it was taken on this grid and layout."""
    path = os.path.join(REPO, "profiles", "r01_leja_traffic.json")
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


def reference_arm(args, rank):
    if rank != 0:
        return
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
    line = {"metric": METRIC, "value": value, "unit": "cell-updates/s", "n_gpus": args.gpus,
            "steps": iters, "warmup": args.warmup, "ms_per_step": 1e3 * args.n ** 2 / value,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE config-1 state: KH 2048^2 + 16 Fourier modes "
                    "per field; v seeded unit Gaussian)", "impl": "reference",
            "config": {"workload": workload_name(args.n), "grid": args.n,
                       "parallelism": "cpu (reference NumPy path: ufuncs on one core, BLAS "
                                      "norms multi-threaded)",
                       "sample": "each step = 1 Leja term (FD-JVP + Newton update + 2 norms) "
                                 "of the alpha*dt=10 call; the metric is per cell-update, so "
                                 "the sweep's rate is the per-term rate"},
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


def main():
    args = parse()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        reference_arm(args, rank)
        return
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2108_13622_b200 as xb
    from paper_2108_13622_b200 import _lib, leja, scenarios as sc

    s = sc.CONFIGS[1]()
    s.nx = s.ny = args.n
    q = sc.initial_fields(s)
    n_cells = s.nx * s.ny
    v_host = sc.unit_gaussian(q.size, s.extra["v_seed"]).reshape(q.shape)
    params = xb.MHDParams(mu=s.mu, eta=s.eta, kappa=s.kappa)
    if world > 1:
        # y-strips: rank r owns rows [y0, y0+ny_r) of the 2048^2 problem (strong scaling)
        from paper_2108_13622_b200 import strips
        comm = strips.Comm()
        mhd = strips.StripMhd(xb.StateGrid(s.nx, s.ny, s.dx, s.dy, None), params, comm)
        _ops_mod = xb.linearize._ops
        _ops_mod.set_reducer(strips.Reducer(comm, torch.device("cuda", local)))
        q_loc = np.ascontiguousarray(mhd.layout.local_rows(q))
        v_loc = np.ascontiguousarray(mhd.layout.local_rows(v_host))
    else:
        mhd = None
        q_loc, v_loc = q, v_host
    u_dev = torch.from_numpy(q_loc).cuda().reshape(-1)
    v_dev = torch.from_numpy(v_loc).cuda().reshape(-1)
    if mhd is None:
        st = xb.StateGrid(s.nx, s.ny, s.dx, s.dy, u_dev.reshape(8, s.ny, s.nx))
        mhd = xb.MhdRhs(st, params)
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

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def maxed(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident timed region
    for _ in range(args.warmup):
        leja._coeff_cache.clear()
        sweep(v_dev)
    stream = torch.cuda.current_stream()
    iters_total = 0
    degrees = None
    launches0 = total_launches(mhd)
    with ClockSampler(local) as clocks:
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            leja._coeff_cache.clear()
            its, outs = sweep(v_dev)
            iters_total += its
            degrees = [r.iterations for r in outs]
        ev1.record(stream)
        barrier()
    launches = total_launches(mhd) - launches0
    ms = maxed(ev0.elapsed_time(ev1))
    # every rank processes its strip of the same iterations: whole-job cell-updates
    value = iters_total * n_cells / (ms * 1e-3)

    # ---- the dominant kernel alone: CUDA events around back-to-back fused iterations
    kern_ms = time_fused_iteration(xb, _lib, lin, mhd, v_dev, alpha)
    # single domain only: in y-strip mode the stencil needs exchanged ghost rows
    stencil_ms = time_stencil_modes(_lib, lin, mhd, v_dev) if world == 1 else {}
    local_cells = u_dev.numel() // 8
    bpc = bytes_per_cell_term(world)
    achieved = bpc * local_cells / (kern_ms * 1e-3) / 1e9
    peak, peak_kind = measured_peaks()

    # ---- end to end through the public API with pinned host buffers
    u_pin = torch.from_numpy(q_loc.reshape(-1)).pin_memory()
    v_pin = torch.from_numpy(v_loc.reshape(-1)).pin_memory()

    def e2e_step():
        its = 0
        leja._coeff_cache.clear()
        op_e = xb.RhsOperator(mhd)
        lin_e = xb.FrozenLinearization(op_e, u_pin)            # H2D u, F(u)
        for adt in SWEEP:
            dt = adt / alpha
            res = xb.apply_phi_leja(1, xb.JacobianAction(lin_e), v_pin, dt,
                                    xb.shift_and_scale(alpha * dt), LEJA_TOL)   # H2D v, D2H p
            assert isinstance(res.vector, np.ndarray)
            its += res.iterations
        return its

    # warm-up of the host side too: the first steps page-lock the result buffers
    # (torch's caching host allocator), which later steps reuse
    for _ in range(args.warmup):
        e2e_step()
    e2e_iters = 0
    barrier()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_iters += e2e_step()
    e1.record(stream)
    barrier()
    e2e_ms = maxed(max(e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t0)))
    vec_bytes = 8 * q.size   # whole job: every rank moves its strip
    e2e = {"value": e2e_iters * n_cells / (e2e_ms * 1e-3), "unit": "cell-updates/s",
           "h2d_bytes_per_step": vec_bytes * (1 + len(SWEEP)),
           "d2h_bytes_per_step": vec_bytes * len(SWEEP)}

    exprb = None
    if not args.no_exprb and rank == 0 and world == 1:
        exprb = exprb_step_time(xb, with_cpu=not args.no_cpu_baseline)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_sample(args.n)

    if rank == 0:
        plan = mhd.ctx.plan()
        line = {
            "metric": METRIC, "value": value, "unit": "cell-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE config-1 state: KH 2048^2 + 16 Fourier modes "
                    "per field; v seeded unit Gaussian)",
            "config": {"workload": workload_name(args.n),
                       "grid": args.n, "alpha": alpha, "leja_degrees": degrees,
                       "l2_policy": "inputs larger than L2 (268 MB per vector)",
                       "parallelism": f"y-strips x{world} (NCCL halo + allreduce)"
                                      if world > 1 else "single-gpu",
                       "stencil_plan": plan},
            "gbs_algorithmic": value * bpc / 1e9,
            "jv_per_s": value / n_cells,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_source": peak_kind,
                         # the same term at the reference's 384 B/cell traffic
                         "frac_at_384B": 384.0 * local_cells / (kern_ms * 1e-3) / 1e9 / peak,
                         "kernel": "stencil_kernel<MODE_LEJA> (fused FD-JVP + Newton update)",
                         "kernel_ms": kern_ms, "bytes_per_cell": bpc,
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
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        if exprb is not None:
            line["exprb_step"] = exprb
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


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
    """Average duration of the fused Leja iteration kernel (CUDA events, same stream)."""
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
                                       int(n_iter), ctypes.byref(out))
    _lib.check(rc, "xmhd_time_leja_iterations")
    torch.cuda.synchronize()
    return float(out.value)


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
