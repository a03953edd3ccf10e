#!/bin/bash
mkdir -p gpurun_out
XMHD_WS=1 timeout 600 python -m pytest tests/test_gpu_ws.py -q -x > gpurun_out/r02j_ws.txt 2>&1; echo "ws rc=$?"; tail -3 gpurun_out/r02j_ws.txt
for v in 1 0; do echo "== XMHD_WS=$v"; XMHD_WS=$v timeout 300 python scripts/prof_leja.py 2048 24 2>&1 | tail -2; done
XMHD_WS=1 timeout 300 python scripts/prof_rhs_jvp.py 2048 > /dev/null 2>&1; echo "rhs/jvp plain rc=$?"
