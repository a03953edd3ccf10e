"""Run a BASELINE.json adaptive configuration end to end on the GPU and report.

    python scripts/run_config.py 0          # KH 128^2, EXPRB43, tol 1e-4, t_end 0.5
    python scripts/run_config.py 2          # double Harris 512^2, EXPRB54s4, tol 1e-6, t_end 10
    python scripts/run_config.py 3          # KH 4096^2, tol 1e-5, 20 adaptive steps
    python scripts/run_config.py 4          # double Harris 8192^2, eta 1e-3, 10 adaptive steps
    torchrun --nproc-per-node 8 scripts/run_config.py 4w   # 16384^2 over 8 GPUs (y-strips)

Prints one JSON line: accepted/rejected steps, RHS evaluations, Leja
iterations, wall seconds (total and per accepted step) and the cell-update rate
of the whole run (RHS evaluations x cells / wall).
"""

import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13622_b200 as xb  # noqa: E402
from paper_2108_13622_b200 import scenarios as sc  # noqa: E402


def strip_comm():
    """Under torchrun (WORLD_SIZE > 1): one rank per GPU over NCCL, the grid in
    y-strips.  XMHD_BENCH_SHARED_GPU=1: the ranks share device 0 over gloo (a
    check of the multi-rank host logic on a one-GPU box, not a measurement)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world == 1:
        return None
    import torch.distributed as dist
    from paper_2108_13622_b200 import strips
    shared = bool(int(os.environ.get("XMHD_BENCH_SHARED_GPU", "0") or "0"))
    local = 0 if shared else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if shared:
        os.environ["XMHD_STRIP_TRANSPORT"] = "nccl"
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return strips.Comm()


def main():
    k = sys.argv[1] if len(sys.argv) > 1 else "0"
    k = int(k) if k.isdigit() else k          # "4w": the 16384^2 weak-scaling case
    comm = strip_comm()
    setup = sc.CONFIGS[k]()
    if len(sys.argv) > 2:
        setup.max_accepted = int(sys.argv[2])
    scheme = xb.Scheme(setup.scheme)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    marks = []

    def on_step(rec, u):
        marks.append(time.perf_counter())

    rep = xb.run(xb.RunConfig(scenario=setup, scheme=scheme, tol=setup.tol,
                              max_accepted=setup.max_accepted), on_step=on_step, comm=comm)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    # per accepted step (host clock at the step's end; the first step also waits
    # for the power-iteration start vector and runs the spectral estimate)
    step_wall = [b - a for a, b in zip(marks, marks[1:])]
    cells = setup.nx * setup.ny
    steps = [s for s in rep.steps if s.accepted]
    out = {"config": k, "name": setup.name, "grid": [setup.nx, setup.ny], "scheme": setup.scheme,
           "tol": setup.tol, "status": rep.status, "accepted": rep.accepted,
           "rejected": rep.rejected, "rhs_evals": rep.rhs_evals,
           "phi_iterations": rep.phi_iterations, "spectrum_rhs_evals": rep.spectrum_rhs_evals,
           "t_reached": rep.t_reached, "wall_s": wall, "run_wall_s": rep.wall_seconds,
           "wall_s_per_step": rep.wall_seconds / max(rep.accepted, 1),
           "wall_s_per_step_after_first": (sum(step_wall) / len(step_wall)) if step_wall else None,
           "step_wall_ms": [round(1e3 * w, 1) for w in step_wall],
           "cell_updates_per_s": rep.rhs_evals * cells / rep.wall_seconds,
           "max_divb": rep.max_divb, "mass_drift": rep.mass_drift,
           "dt_first_last": [steps[0].dt, steps[-1].dt] if steps else None,
           "checksum": rep.checksum}
    if comm is not None:
        out["ranks"] = comm.size
    if comm is None or comm.rank == 0:
        print(json.dumps(out), flush=True)
    if comm is not None:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
