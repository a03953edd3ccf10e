# source-level ncu capture of the two fused Leja term variants (PM_LOOK, PM_SKIP) at 2048^2
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel --launch-skip 2 -c 2 -o gpurun_out/g2_leja python scripts/prof_leja.py 2048 3 > gpurun_out/g2_ncu.log 2>&1
for v in build/ab_*.so; do [ -f "$v" ] || continue; for n in 2048 4096; do XMHD_SO=$v timeout 120 python scripts/prof_leja.py $n 40 >> gpurun_out/g2_ab_$(basename $v .so).log 2>&1; done; done
for n in 2048 4096; do timeout 120 python scripts/prof_leja.py $n 40 >> gpurun_out/g2_ab_base.log 2>&1; done
