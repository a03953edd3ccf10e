for k in 0 2 3 4; do timeout 900 python scripts/run_config.py $k 2>&1 | grep '^{' >> gpurun_out/r1s3l_configs.jsonl; done
