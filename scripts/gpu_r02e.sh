#!/bin/bash
# r02: warp-specialized TMA kernel -- bitwise vs the one-role kernel, the GPU
# suite, then an A/B of the bench (XMHD_WS=0 = one-role kernel)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ws.py -q -x > gpurun_out/r02e_ws.txt 2>&1; echo "ws rc=$?"; tail -15 gpurun_out/r02e_ws.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02e_pytest.txt 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r02e_pytest.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-exprb > gpurun_out/r02e_bench_ws.json 2> gpurun_out/r02e_bench_ws.err; echo "bench ws rc=$?"
XMHD_WS=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-exprb --no-scale-case > gpurun_out/r02e_bench_one.json 2> gpurun_out/r02e_bench_one.err; echo "bench one rc=$?"
python - <<'PY'
import json
for tag in ("ws", "one"):
    try:
        d = json.loads(open(f"gpurun_out/r02e_bench_{tag}.json").read())
    except Exception as e:
        print(tag, "no line", e); continue
    r = d["roofline"]
    print(tag, "value %.3e" % d["value"], "ms/step %.1f" % d["ms_per_step"], "kernel_ms %.4f" % r["kernel_ms"], "frac %.3f" % r["frac"],
          {k: round(v["kernel_ms"], 4) for k, v in (r.get("by_kind") or {}).items()},
          {k: round(v["kernel_ms"], 4) for k, v in d.get("stencil_kernels", {}).items()}, d["clocks"].get("sm_mhz"),
          "scale", d.get("scale_case", {}).get("value"))
PY
