#!/bin/bash
# r02 checkpoint: full GPU suite, smoke, the bench as the driver runs it, reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02n_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02n_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02n_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02n_smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02n_bench.json").read())
r = d["roofline"]
print("value %.4e ms/step %.1f kernel_ms %.4f frac %.3f" % (d["value"], d["ms_per_step"], r["kernel_ms"], r["frac"]),
      {k: (round(v["kernel_ms"], 4), round(v["frac"], 3)) for k, v in (r.get("by_kind") or {}).items()},
      "e2e %.3e pinned %.3e" % (d["e2e"]["value"], d["e2e_pinned"]["value"]), d["clocks"],
      "scale", d.get("scale_case", {}).get("value"), "exprb", d.get("exprb_step", {}).get("wall_s_per_step"),
      "cpu", d.get("cpu_baseline", {}).get("value"))
PY
