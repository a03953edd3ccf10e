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
