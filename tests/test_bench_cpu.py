"""bench.py host-side pieces that run without a GPU: the clock sampler's
summary (throttle reasons the timing rules reject or note) from both sample
sources."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def test_clock_summary_parses_nvml_and_smi_lines():
    c = bench.ClockSampler(0)
    c.lines = ["1830, 1965, 0, Not Active, Not Active, Not Active, Active",     # NVML sampler
               "1875, 1965, 0, Not Active, Not Active, Not Active, Not Active",
               "1700, 1965, 612.5, Not Active, Active, Not Active, Active",      # nvidia-smi csv
               "garbage"]
    s = c.summary()
    assert s["samples"] == 3
    assert s["sm_mhz"] == 1830.0 and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["hw_thermal_slowdown", "sw_power_cap"]


def test_clock_sampler_without_gpu_is_empty():
    with bench.ClockSampler(0) as c:
        pass
    assert c.summary()["samples"] >= 0


def test_multi_gpu_request_without_gpus_fails_loudly():
    """`bench.py --gpus 2` must never time one GPU and report it as two: with
    fewer visible GPUs it exits non-zero with a message."""
    import subprocess
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(bench.__file__), "bench.py"),
                        "--gpus", "2", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2
    assert "refusing" in r.stderr
    assert r.stdout.strip() == ""


def test_both_arms_share_the_config_dict():
    assert bench.workload_config(2048) == bench.workload_config(2048)
    cfg = bench.workload_config(2048)
    assert cfg["grid"] == 2048 and cfg["alpha_dt"] == list(bench.SWEEP)
