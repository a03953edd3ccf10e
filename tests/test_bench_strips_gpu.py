"""bench.py's N>1 path end to end on the one GPU of the test box: the ranks share
device 0 over gloo (XMHD_BENCH_SHARED_GPU=1: torch.distributed strip transport,
point-to-point messages staged through the host, no kernel waits on a peer).
Not a measurement: it checks that every leg of the multi-rank bench runs
(strip set-up from the rank's own rows, the phi sweep, the end-to-end legs, the
8192^2-style scale case on a smaller grid) and agrees with the one-rank run.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(gpus, extra_env):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    env.update(extra_env)
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", str(gpus),
                        "--steps", "1", "--warmup", "1", "--n", "1536", "--scale-n", "1536",
                        "--no-exprb", "--no-cpu-baseline"],
                       capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_multi_rank_bench_path_runs_and_agrees_with_one_rank():
    one = _bench(1, {})
    assert one["n_gpus"] == 1 and "dry_run" not in one
    assert one["roofline"]["share_of_step"] > 0.5
    for n in (2, 3):
        d = _bench(n, {"XMHD_BENCH_SHARED_GPU": "1"})
        assert d["n_gpus"] == n and "not a measurement" in d["dry_run"]
        assert d["parallelism"].startswith(f"y-strips x{n} (NCCL")
        assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
        # the same phi-actions: spectral estimate and degrees of the one-rank run
        # (low degrees exactly; the long calls may move by a term with the
        # summation order of the norms)
        assert abs(d["workload_detail"]["alpha"] / one["workload_detail"]["alpha"] - 1) < 1e-9
        got, want = d["workload_detail"]["leja_degrees"], one["workload_detail"]["leja_degrees"]
        assert got[:2] == want[:2]
        assert all(abs(a - b) <= 2 for a, b in zip(got, want))
        sc_n, sc_1 = d["scale_case"], one["scale_case"]
        assert sc_n["n_gpus"] == n and sc_n["leja_degrees"][:2] == sc_1["leja_degrees"][:2]
        assert d["roofline"]["kernel_ms_alone"] is None and d["roofline"]["frac"] > 0


def _run_config(args, ranks):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    script = os.path.join(REPO, "scripts", "run_config.py")
    if ranks == 1:
        cmd = [sys.executable, script] + args
    else:
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        env["XMHD_BENCH_SHARED_GPU"] = "1"
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={ranks}", "--master-addr", "127.0.0.1", "--master-port",
               str(port), script] + args
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_adaptive_run_over_real_ranks_keeps_the_counters():
    """harness.run over y-strips with one process per rank (torch.distributed
    Comm, each rank its own rows of the initial state and of the start vector):
    the one-rank run's accept / reject sequence, RHS and Leja counts."""
    one = _run_config(["2", "8"], 1)
    assert one["accepted"] == 8 and one.get("ranks") is None
    for n in (2, 3):
        d = _run_config(["2", "8"], n)
        assert d["ranks"] == n
        for key in ("accepted", "rejected", "rhs_evals", "phi_iterations", "spectrum_rhs_evals"):
            assert d[key] == one[key], key
        assert abs(d["t_reached"] / one["t_reached"] - 1) < 1e-6
        assert abs(d["max_divb"] - one["max_divb"]) <= 1e-9 * max(1.0, abs(one["max_divb"]))
