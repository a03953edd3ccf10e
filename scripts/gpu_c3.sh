timeout 600 python -m pytest tests/test_gpu_async.py -q > gpurun_out/r1s2j_async.log 2>&1; echo "rc=$?" >> gpurun_out/r1s2j_async.log
timeout 600 python scripts/prof_timeline.py c3 5 2>&1 | grep -v Warn > gpurun_out/r1s2j_tl_c3.log
