#!/bin/bash
# native staged H2D sweep + vector-kernel bandwidths
mkdir -p gpurun_out
nproc
for cfg in "XMHD_H2D_PY=1" "XMHD_H2D_THREADS=4" "XMHD_H2D_THREADS=6" "XMHD_H2D_THREADS=8" "XMHD_H2D_THREADS=12" "XMHD_H2D_THREADS=16" \
           "XMHD_H2D_THREADS=8 XMHD_H2D_NT=0" "XMHD_H2D_THREADS=12 XMHD_H2D_NT=0" "XMHD_H2D_THREADS=8 XMHD_H2D_CHUNK_MB=8" "XMHD_H2D_THREADS=8 XMHD_H2D_CHUNK_MB=32" \
           "XMHD_H2D_THREADS=8 XMHD_H2D_CHUNK_MB=4 XMHD_H2D_SLOTS=8" ""; do
  env $cfg timeout 120 python scripts/probe_h2d_native.py 2>&1 | tail -1
done | tee gpurun_out/r02q_h2d.txt
timeout 300 python scripts/prof_vec.py 4096 2>&1 | tee gpurun_out/r02q_vec.txt
timeout 300 python scripts/probe_h2d.py 2>&1 | tee gpurun_out/r02q_h2d_py.txt
