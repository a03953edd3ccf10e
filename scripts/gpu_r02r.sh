#!/bin/bash
# fused stage algebra / zero-copy Leja calls / vectorised stream kernels: tests, then timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused_algebra.py -m gpu -q -x > gpurun_out/r02r_new.txt 2>&1; echo "new tests rc=$?"; tail -15 gpurun_out/r02r_new.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02r_pytest.txt 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r02r_pytest.txt
timeout 300 python scripts/prof_vec.py 4096 2>&1 | tee gpurun_out/r02r_vec.txt
timeout 600 python scripts/prof_timeline.py c4 3 > gpurun_out/r02r_timeline_c4.txt 2>&1; echo "timeline rc=$?"; tail -22 gpurun_out/r02r_timeline_c4.txt
timeout 600 python scripts/run_config.py 4 10 2>&1 | tail -3
timeout 600 python scripts/run_config.py 3 20 2>&1 | tail -3
