timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r1s3f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1s3f_pytest.log
for i in 1 2 3; do timeout 200 python scripts/prof_host.py c0 2>&1 | head -1 >> gpurun_out/r1s3f_c0.log; done
timeout 300 python scripts/prof_host.py c2 2>&1 | head -1 >> gpurun_out/r1s3f_c0.log
