timeout 300 python scripts/prof_sweep.py > gpurun_out/r1s3b_sweep.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r1s3b_bench.json 2> gpurun_out/r1s3b_bench.err
timeout 600 python bench.py --no-cpu-baseline --no-exprb --steps 6 > gpurun_out/r1s3b_bench6.json 2>> gpurun_out/r1s3b_bench.err
