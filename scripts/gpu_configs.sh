timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r1s3a_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1s3a_pytest.log
for k in 3 4; do timeout 900 python scripts/run_config.py $k 2>&1 | grep '^{' >> gpurun_out/r1s3a_configs.jsonl; done
