timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r1s3c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1s3c_pytest.log
timeout 200 python scripts/prof_host.py c0 2>&1 | head -1 > gpurun_out/r1s3c_c0.log
timeout 200 python scripts/prof_host.py c0 2>&1 | head -1 >> gpurun_out/r1s3c_c0.log
timeout 300 python scripts/prof_host.py c2 2>&1 | head -1 >> gpurun_out/r1s3c_c0.log
timeout 300 python scripts/prof_timeline.py c0 2>&1 | grep -v Warn > gpurun_out/r1s3c_tl_c0.log
