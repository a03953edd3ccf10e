#!/bin/bash
# final r02 pass: full GPU suite, smoke, bench as the driver runs it, reference arm,
# ncu launch list of the bench command, full ncu captures of the stencil kernels
mkdir -p gpurun_out
T=r03f
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${T}_smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_reference_arm.json 2> gpurun_out/${T}_reference_arm.err; echo "reference rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r03f_bench.json").read())
r = d["roofline"]
print("value %.4e ms/step %.1f kernel_ms %.4f frac %.3f" % (d["value"], d["ms_per_step"], r["kernel_ms"], r["frac"]),
      {k: (round(v["kernel_ms"], 4), round(v["frac"], 3)) for k, v in (r.get("by_kind") or {}).items()},
      "e2e %.3e pinned %.3e" % (d["e2e"]["value"], d["e2e_pinned"]["value"]), d["clocks"],
      "scale", d.get("scale_case", {}).get("value"), "exprb", d.get("exprb_step", {}).get("wall_s_per_step"),
      "c2", d.get("exprb_step_c2", {}).get("wall_s_per_step"), "cpu", d.get("cpu_baseline", {}).get("value"),
      "stencils", {k: (round(v["kernel_ms"], 4), round(v["frac"], 3)) for k, v in d["stencil_kernels"].items()})
PY
# launch list of the bench command (cold, serialised: shares only)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-exprb --no-scale-case > gpurun_out/${T}_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
python scripts/launch_summary.py gpurun_out/${T}_launches.csv "bench.py --steps 2 --warmup 1 (no cpu / exprb / scale legs)" > gpurun_out/${T}_bench_launches.txt 2>&1; head -12 gpurun_out/${T}_bench_launches.txt
# full captures: the two Leja term kinds, RHS, JVP at 2048^2 (config-1 state)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel --launch-skip 3 -c 2 -o gpurun_out/${T}_leja python scripts/prof_leja.py 2048 5 > gpurun_out/${T}_ncu_leja.log 2>&1; echo "ncu leja rc=$?"
python scripts/ncu_summary.py gpurun_out/${T}_leja.ncu-rep "r03 final: fused Leja term, 2048^2 config-1 state, two consecutive launches" > gpurun_out/${T}_leja_ncu.txt 2>&1
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"stencil_kernel<.int.0" --launch-skip 1 -c 1 -o gpurun_out/${T}_rhs python scripts/prof_rhs_jvp.py 2048 > gpurun_out/${T}_ncu_rhs.log 2>&1; echo "ncu rhs rc=$?"
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"stencil_kernel<.int.1" --launch-skip 1 -c 1 -o gpurun_out/${T}_jvp python scripts/prof_rhs_jvp.py 2048 > gpurun_out/${T}_ncu_jvp.log 2>&1; echo "ncu jvp rc=$?"
python scripts/ncu_summary.py gpurun_out/${T}_rhs.ncu-rep "r03 final: RHS stencil, 2048^2" > gpurun_out/${T}_rhs_jvp_ncu.txt 2>&1
python scripts/ncu_summary.py gpurun_out/${T}_jvp.ncu-rep "r03 final: FD-JVP stencil, 2048^2" >> gpurun_out/${T}_rhs_jvp_ncu.txt 2>&1
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"lincomb_kernel" --launch-skip 3 -c 1 -o gpurun_out/${T}_lincomb python scripts/prof_vec.py 4096 > gpurun_out/${T}_ncu_vec.log 2>&1; echo "ncu vec rc=$?"
python scripts/ncu_summary.py gpurun_out/${T}_lincomb.ncu-rep "r03 final: lincomb (2 terms), n = 1.3e8" > gpurun_out/${T}_lincomb_ncu.txt 2>&1
tail -30 gpurun_out/${T}_leja_ncu.txt
# the reports stay on the box except the Leja one (gpurun_out is limited to 64 MiB)
rm -f gpurun_out/${T}_rhs.ncu-rep gpurun_out/${T}_jvp.ncu-rep gpurun_out/${T}_lincomb.ncu-rep
