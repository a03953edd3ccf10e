#!/bin/bash
# r02: full GPU suite (incl. the large-size reference fixtures), the bench as
# the driver runs it, its launch list, and one ncu capture of the fused term
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r02g_pytest.txt 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r02g_pytest.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02g_ref.json 2> gpurun_out/r02g_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02g_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-exprb --no-scale-case > gpurun_out/r02g_ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel --launch-skip 2 -c 2 -o gpurun_out/r02g_leja python scripts/prof_leja.py 2048 3 > gpurun_out/r02g_ncu.log 2>&1; echo "ncu full rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02g_bench.json").read())
r = d["roofline"]
print("value %.4e ms/step %.1f kernel_ms %.4f frac %.3f" % (d["value"], d["ms_per_step"], r["kernel_ms"], r["frac"]),
      {k: (round(v["kernel_ms"], 4), round(v["frac"], 3)) for k, v in (r.get("by_kind") or {}).items()},
      "e2e %.3e pinned %.3e" % (d["e2e"]["value"], d["e2e_pinned"]["value"]), d["clocks"],
      "scale", d.get("scale_case", {}).get("value"), d.get("scale_case", {}).get("ms_per_step"))
PY
