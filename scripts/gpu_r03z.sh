#!/bin/bash
# closing check of the final code: full GPU suite, smoke, the bench as the driver runs it
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r03z_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r03z_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r03z_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r03z_smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r03z_bench.json 2> gpurun_out/r03z_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r03z_bench.json").read())
r = d["roofline"]
print("steps", d["steps"], "value %.4e ms/step %.1f kernel_ms %.4f frac %.3f share %.3f alone %.4f" % (d["value"], d["ms_per_step"], r["kernel_ms"], r["frac"], r["share_of_step"], r["kernel_ms_alone"]),
      {k: (round(v["kernel_ms"], 4), round(v["frac"], 3)) for k, v in (r.get("by_kind") or {}).items()},
      "e2e %.3e pinned %.3e" % (d["e2e"]["value"], d["e2e_pinned"]["value"]), d["clocks"],
      "scale", d.get("scale_case", {}).get("value"), "exprb", d.get("exprb_step", {}).get("wall_s_per_step"),
      "c2", d.get("exprb_step_c2", {}).get("wall_s_per_step"), "cpu", d.get("cpu_baseline", {}).get("value"),
      "stencils", {k: (round(v["kernel_ms"], 4), round(v["frac"], 3)) for k, v in d["stencil_kernels"].items()})
PY
timeout 600 python scripts/run_config.py 4 10 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['accepted'], d['rhs_evals'], d['phi_iterations'], round(d['wall_s_per_step'],4), 'after first', round(d['wall_s_per_step_after_first'],4), d['checksum'][:12])"
timeout 600 python scripts/run_config.py 3 20 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['accepted'], d['rhs_evals'], d['phi_iterations'], round(d['wall_s_per_step'],4), 'after first', round(d['wall_s_per_step_after_first'],4), d['checksum'][:12])"
timeout 600 python scripts/run_config.py 2 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['accepted'], d['rhs_evals'], d['phi_iterations'], round(d['wall_s_per_step'],5), d['checksum'][:12])"
timeout 600 python scripts/run_config.py 0 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['accepted'], d['rhs_evals'], d['phi_iterations'], round(d['wall_s_per_step'],5), d['checksum'][:12])"
