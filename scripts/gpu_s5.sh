# session-5 GPU pass: sweep diagnosis, the default bench twice, configs 3/4
# with the parallel start-vector draw, the GPU suite.
timeout 600 python scripts/diag_sweep.py 4 > gpurun_out/s5_diag.jsonl 2> gpurun_out/s5_diag.err
timeout 900 python bench.py > gpurun_out/s5_bench1.json 2> gpurun_out/s5_bench.err
timeout 900 python bench.py > gpurun_out/s5_bench2.json 2>> gpurun_out/s5_bench.err
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s5_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s5_pytest.log
for k in 3 4; do timeout 900 python scripts/run_config.py $k 2>&1 | grep '^{' >> gpurun_out/s5_configs.jsonl; done
nproc > gpurun_out/s5_host.txt; lscpu | head -20 >> gpurun_out/s5_host.txt
