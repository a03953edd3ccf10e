#!/bin/bash
# ncu of the RHS stencil with 3 CTAs per SM (166 registers, no spills, 70 KB rings) against the default build
mkdir -p gpurun_out
T=r03c
timeout 300 python scripts/prof_rhs_jvp.py 2048 > /dev/null 2>&1
for V in default build/ab_ring3m3.so; do
  N=$(basename $V .so)
  if [ $V = default ]; then unset XMHD_SO; else export XMHD_SO=$V; fi
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"stencil_kernel<.int.0" --launch-skip 1 -c 1 -o gpurun_out/${T}_rhs_$N python scripts/prof_rhs_jvp.py 2048 > gpurun_out/${T}_ncu_$N.log 2>&1; echo "ncu $N rc=$?"
done
