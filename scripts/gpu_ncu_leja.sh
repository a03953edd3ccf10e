# full ncu capture (source-level) of the two fused Leja term variants at 2048^2
# usage: bash scripts/gpu_ncu_leja.sh TAG
tag=$1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel --launch-skip 2 -c 2 -o gpurun_out/${tag}_leja python scripts/prof_leja.py 2048 3 > gpurun_out/${tag}_ncu.log 2>&1
