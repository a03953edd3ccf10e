timeout 600 python -m pytest tests/test_gpu_async.py -q > gpurun_out/r1s2e_async.log 2>&1; echo "rc=$?" >> gpurun_out/r1s2e_async.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r1s2e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1s2e_pytest.log
timeout 300 python scripts/prof_host.py c2 1.0 > gpurun_out/r1s2e_host_c2.log 2>&1
echo done
