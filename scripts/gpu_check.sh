timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r1s2o_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1s2o_pytest.log
timeout 300 python scripts/prof_sweep.py > gpurun_out/r1s2o_sweep.log 2>&1
timeout 600 python bench.py > gpurun_out/r1s2o_bench.json 2> gpurun_out/r1s2o_bench.err
timeout 600 python bench.py --no-cpu-baseline --no-exprb > gpurun_out/r1s2o_bench2.json 2>> gpurun_out/r1s2o_bench.err
