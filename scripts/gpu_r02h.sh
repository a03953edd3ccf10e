#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_large_parity.py -q > gpurun_out/r02h_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02h_pytest.txt
timeout 300 python scripts/prof_rhs_jvp.py 2048 > gpurun_out/r02h_plain.txt 2>&1; echo "plain rc=$?"
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"stencil_kernel<0" --launch-skip 1 -c 1 -o gpurun_out/r02h_rhs python scripts/prof_rhs_jvp.py 2048 > gpurun_out/r02h_ncu_rhs.log 2>&1; echo "ncu rhs rc=$?"
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"stencil_kernel<1" --launch-skip 1 -c 1 -o gpurun_out/r02h_jvp python scripts/prof_rhs_jvp.py 2048 > gpurun_out/r02h_ncu_jvp.log 2>&1; echo "ncu jvp rc=$?"
