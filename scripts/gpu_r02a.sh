#!/bin/bash
# r02 first pass: GPU tests, fp64 ceilings, a short bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02a_smi.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/r02a_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r02a_pytest.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak scripts/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/r02a_fp64.jsonl 2>&1
python bench.py --steps 5 --warmup 3 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/r02a_pytest.txt; cat gpurun_out/r02a_fp64.jsonl
