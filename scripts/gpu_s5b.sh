# session-5 pass 2: start-vector wait probes (configs 3/4), strips-off GPU edge tests, bench.
timeout 600 python -m pytest tests/test_gpu_edge.py -q -k prefetched > gpurun_out/s5b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s5b_pytest.log
for k in 3 4; do timeout 900 python scripts/probe_rng_wait.py $k > gpurun_out/s5b_rngwait_c$k.log 2>&1; done
timeout 900 python bench.py > gpurun_out/s5b_bench.json 2> gpurun_out/s5b_bench.err
