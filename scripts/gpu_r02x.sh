#!/bin/bash
mkdir -p gpurun_out
T=r02x
timeout 300 python scripts/probe_call_host.py 4096 2>&1 | tail -6
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"stencil_kernel<.int.0," --launch-skip 1 -c 1 -o gpurun_out/${T}_rhs python scripts/prof_rhs_jvp.py 2048 > gpurun_out/${T}_ncu_rhs.log 2>&1; echo "ncu rhs rc=$?"
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"stencil_kernel<.int.1," --launch-skip 1 -c 1 -o gpurun_out/${T}_jvp python scripts/prof_rhs_jvp.py 2048 > gpurun_out/${T}_ncu_jvp.log 2>&1; echo "ncu jvp rc=$?"
python scripts/ncu_summary.py gpurun_out/${T}_rhs.ncu-rep "r02 final: RHS stencil, 2048^2" > gpurun_out/${T}_rhs_jvp_ncu.txt 2>&1
python scripts/ncu_summary.py gpurun_out/${T}_jvp.ncu-rep "r02 final: FD-JVP stencil, 2048^2" >> gpurun_out/${T}_rhs_jvp_ncu.txt 2>&1
cat gpurun_out/${T}_rhs_jvp_ncu.txt | grep -v "^$" | head -50
for th in 8 12 8 12; do
XMHD_H2D_THREADS=$th timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-exprb --no-scale-case > gpurun_out/${T}_bench_$th.json 2> gpurun_out/${T}_bench_$th.err
python - <<PY
import json
d = json.loads(open("gpurun_out/${T}_bench_$th.json").read())
print("threads $th value %.4e ms/step %.1f" % (d["value"], d["ms_per_step"]), "e2e %.3e (%.1f ms) pinned %.3e (%.1f ms)" % (d["e2e"]["value"], d["e2e"]["ms_per_step"], d["e2e_pinned"]["value"], d["e2e_pinned"]["ms_per_step"]), d["clocks"]["sm_mhz"])
PY
done
