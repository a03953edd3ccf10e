timeout 600 python -m pytest tests/test_gpu_async.py -q -x > gpurun_out/r1s2x_async.log 2>&1; echo "rc=$?" >> gpurun_out/r1s2x_async.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r1s2x_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1s2x_pytest.log
timeout 200 python scripts/prof_host.py c0 2>&1 | head -1 > gpurun_out/r1s2x_c0.log
XMHD_NATIVE_STEP=0 timeout 200 python scripts/prof_host.py c0 2>&1 | head -1 >> gpurun_out/r1s2x_c0.log
timeout 300 python scripts/prof_host.py c2 2>&1 | head -1 >> gpurun_out/r1s2x_c0.log
timeout 300 python scripts/prof_timeline.py c0 2>&1 | grep -v Warn > gpurun_out/r1s2x_tl_c0.log
