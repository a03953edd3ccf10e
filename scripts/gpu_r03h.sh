#!/bin/bash
# N>1 bench path on the one GPU: ranks share device 0 over gloo (host-logic check, not a measurement)
mkdir -p gpurun_out
for N in 2 3; do
XMHD_BENCH_SHARED_GPU=1 timeout 1200 python bench.py --gpus $N --steps 1 --warmup 1 > gpurun_out/r03h_bench_$N.json 2> gpurun_out/r03h_bench_$N.err; echo "N=$N rc=$?"
tail -5 gpurun_out/r03h_bench_$N.err
python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/r03h_bench_$N.json").read().strip().splitlines()[-1])
    print({k: d.get(k) for k in ("n_gpus", "value", "ms_per_step", "parallelism", "dry_run", "gpu_launches")})
    print(d["workload_detail"]); print(d["roofline"]["kernel_ms"], d["roofline"]["timed"]); print(d.get("scale_case"))
    print(d["e2e"])
except Exception as e:
    print("no line:", e)
PY
done
