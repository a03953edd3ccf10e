#!/bin/bash
mkdir -p gpurun_out
for cfg in "" "XMHD_H2D_THREADS=6" "XMHD_H2D_THREADS=12"; do env $cfg timeout 120 python scripts/probe_h2d_native.py 2>&1 | tail -1; done
for k in 1 2 3; do
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-exprb --no-scale-case > gpurun_out/r02u_bench_$k.json 2> gpurun_out/r02u_bench_$k.err; echo "bench rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/r02u_bench_$k.json").read())
r = d["roofline"]
print("value %.4e ms/step %.1f kernel_ms %.4f frac %.3f" % (d["value"], d["ms_per_step"], r["kernel_ms"], r["frac"]),
      "e2e %.3e (%.1f ms) pinned %.3e (%.1f ms)" % (d["e2e"]["value"], d["e2e"]["ms_per_step"], d["e2e_pinned"]["value"], d["e2e_pinned"]["ms_per_step"]), d["clocks"]["sm_mhz"])
PY
done
timeout 600 python scripts/run_config.py 4 10 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['accepted'], d['rhs_evals'], d['phi_iterations'], round(d['wall_s_per_step'],4), d['checksum'][:16])"
timeout 600 python scripts/run_config.py 3 20 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['accepted'], d['rhs_evals'], d['phi_iterations'], round(d['wall_s_per_step'],4), d['checksum'][:16])"

