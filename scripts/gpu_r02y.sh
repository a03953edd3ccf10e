#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_capi_only.py tests/test_gpu_fused_algebra.py -m gpu -q -x > gpurun_out/r02y_capi.txt 2>&1; echo "capi rc=$?"; tail -15 gpurun_out/r02y_capi.txt
for k in 1 2; do
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-exprb --no-scale-case > gpurun_out/r02y_bench_$k.json 2> gpurun_out/r02y_bench_$k.err
python - <<PY
import json
d = json.loads(open("gpurun_out/r02y_bench_$k.json").read())
print("value %.4e ms/step %.1f kernel %.4f" % (d["value"], d["ms_per_step"], d["roofline"]["kernel_ms"]), "e2e %.3e (%.1f ms) pinned %.3e (%.1f ms)" % (d["e2e"]["value"], d["e2e"]["ms_per_step"], d["e2e_pinned"]["value"], d["e2e_pinned"]["ms_per_step"]), d["clocks"]["sm_mhz"])
PY
done
