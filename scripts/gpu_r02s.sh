#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused_algebra.py -m gpu -q -x > gpurun_out/r02s_new.txt 2>&1; echo "new tests rc=$?"; tail -3 gpurun_out/r02s_new.txt
timeout 600 python scripts/probe_degrees.py 4 6 2>&1 | tail -1
timeout 600 python scripts/probe_degrees.py 3 20 2>&1 | tail -1
timeout 600 python scripts/prof_timeline.py c4 4 > gpurun_out/r02s_timeline_c4.txt 2>&1; echo "timeline rc=$?"; grep -A16 "steady state" gpurun_out/r02s_timeline_c4.txt
timeout 600 python scripts/prof_timeline.py c3 8 > gpurun_out/r02s_timeline_c3.txt 2>&1; echo "timeline rc=$?"; grep -B14 -A16 "steady state" gpurun_out/r02s_timeline_c3.txt | tail -45
XMHD_FUSE_STAGES=0 XMHD_ZERO_COPY=0 timeout 600 python scripts/run_config.py 3 20 2>&1 | tail -1 | cut -c1-200
XMHD_FUSE_STAGES=0 XMHD_ZERO_COPY=0 timeout 600 python scripts/run_config.py 3 20 2>&1 | tail -1 | grep -o '"checksum": "[0-9a-f]*"'
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02s_bench.json 2> gpurun_out/r02s_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02s_bench.json").read())
r = d["roofline"]
print("value %.4e ms/step %.1f kernel_ms %.4f frac %.3f" % (d["value"], d["ms_per_step"], r["kernel_ms"], r["frac"]),
      {k: (round(v["kernel_ms"], 4), round(v["frac"], 3)) for k, v in (r.get("by_kind") or {}).items()},
      "e2e %.3e pinned %.3e" % (d["e2e"]["value"], d["e2e_pinned"]["value"]), d["clocks"],
      "scale", d.get("scale_case", {}).get("value"), "exprb", d.get("exprb_step", {}).get("wall_s_per_step"),
      "c2", d.get("exprb_step_c2", {}).get("wall_s_per_step"), "cpu", d.get("cpu_baseline", {}).get("value"))
PY
