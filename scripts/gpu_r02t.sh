#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused_algebra.py -m gpu -q -x > gpurun_out/r02t_new.txt 2>&1; echo "new tests rc=$?"; tail -12 gpurun_out/r02t_new.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02t_pytest.txt 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02t_pytest.txt
for ad in 0 1; do
  echo "== XMHD_ADAPTIVE=$ad"
  XMHD_ADAPTIVE=$ad timeout 600 python scripts/run_config.py 4 10 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['accepted'], d['rhs_evals'], d['phi_iterations'], round(d['wall_s_per_step'],4), d['checksum'][:16])"
  XMHD_ADAPTIVE=$ad timeout 600 python scripts/run_config.py 3 20 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['accepted'], d['rhs_evals'], d['phi_iterations'], round(d['wall_s_per_step'],4), d['checksum'][:16])"
done
timeout 600 python scripts/prof_timeline.py c4 4 > gpurun_out/r02t_timeline_c4.txt 2>&1; echo "timeline rc=$?"; grep -B17 -A16 "steady state" gpurun_out/r02t_timeline_c4.txt
timeout 600 python scripts/prof_timeline.py c3 8 > gpurun_out/r02t_timeline_c3.txt 2>&1; echo "timeline rc=$?"; grep -A12 "steady state" gpurun_out/r02t_timeline_c3.txt
for ad in 0 1; do
XMHD_ADAPTIVE=$ad timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-exprb > gpurun_out/r02t_bench_$ad.json 2> gpurun_out/r02t_bench_$ad.err; echo "bench rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/r02t_bench_$ad.json").read())
r = d["roofline"]
print("value %.4e ms/step %.1f kernel_ms %.4f frac %.3f" % (d["value"], d["ms_per_step"], r["kernel_ms"], r["frac"]),
      "e2e %.3e pinned %.3e" % (d["e2e"]["value"], d["e2e_pinned"]["value"]), d["clocks"]["sm_mhz"],
      "scale", d.get("scale_case", {}).get("value"), "launches", d["gpu_launches"])
PY
done
