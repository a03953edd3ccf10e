#!/bin/bash
# in-region term timing: its test, then the bench as the driver runs it (twice: box state)
mkdir -p gpurun_out
T=r03g
timeout 900 python -m pytest tests/test_gpu_fused_algebra.py tests/test_capi_only.py -m gpu -q -x 2>&1 | tail -3
for k in 1 2; do
timeout 900 python bench.py > gpurun_out/${T}_bench_$k.json 2> gpurun_out/${T}_bench_$k.err; echo "bench rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/${T}_bench_$k.json").read())
r = d["roofline"]
print("steps", d["steps"], "value %.4e ms/step %.1f kernel_ms %.4f frac %.3f share %.3f alone %.4f frac_alone %.3f" % (d["value"], d["ms_per_step"], r["kernel_ms"], r["frac"], r["share_of_step"], r["kernel_ms_alone"], r["frac_alone"]),
      {k: (round(v["kernel_ms"], 4), round(v["frac"], 3)) for k, v in (r.get("by_kind") or {}).items()},
      "e2e %.3e pinned %.3e" % (d["e2e"]["value"], d["e2e_pinned"]["value"]), d["clocks"],
      "scale", d.get("scale_case", {}).get("value"), "exprb", d.get("exprb_step", {}).get("wall_s_per_step"),
      "c2", d.get("exprb_step_c2", {}).get("wall_s_per_step"), "cpu", d.get("cpu_baseline", {}).get("value"),
      "stencils", {k: (round(v["kernel_ms"], 4), round(v["frac"], 3)) for k, v in d["stencil_kernels"].items()})
PY
done
