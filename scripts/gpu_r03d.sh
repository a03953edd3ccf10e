#!/bin/bash
# RHS kernel with the ideal y-fluxes in registers (default build) vs the shared-memory ring (-DXB_FYREG=0);
# verified peer link / NCCL fallback test
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_peer_ipc_gpu.py tests/test_gpu_edge.py -m gpu -q -x 2>&1 | tail -3
for rep in 1 2 3; do
for n in 2048 4096; do
timeout 300 python scripts/prof_modes.py $n 2>&1 | grep "RHS"
XMHD_SO=build/ab_nofyreg.so timeout 300 python scripts/prof_modes.py $n 2>&1 | grep "RHS" | sed 's/^/   ring: /'
done
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"stencil_kernel<.int.0" --launch-skip 1 -c 1 -o gpurun_out/r03d_rhs_fyreg python scripts/prof_rhs_jvp.py 2048 > gpurun_out/r03d_ncu.log 2>&1; echo "ncu rc=$?"
