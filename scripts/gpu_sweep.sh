timeout 300 python scripts/prof_sweep.py > gpurun_out/r1s2n_sweep.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r1s2n_bench.json 2> gpurun_out/r1s2n_bench.err
