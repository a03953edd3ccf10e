timeout 600 python -m pytest tests/test_gpu_async.py -x -q > gpurun_out/r1s2d_async.log 2>&1; echo "rc=$?" >> gpurun_out/r1s2d_async.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r1s2d_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1s2d_pytest.log
timeout 200 python scripts/prof_host.py c0 > gpurun_out/r1s2d_host_c0.log 2>&1
timeout 300 python scripts/prof_timeline.py c0 > gpurun_out/r1s2d_tl_c0.log 2>&1
timeout 300 python scripts/prof_timeline.py c2 1.0 > gpurun_out/r1s2d_tl_c2.log 2>&1
echo done
