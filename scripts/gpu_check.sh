timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r1s2w_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1s2w_pytest.log
timeout 200 python scripts/prof_tile.py 128 512 > gpurun_out/r1s2w_tile.log 2>&1
timeout 200 python scripts/prof_host.py c0 2>&1 | head -1 > gpurun_out/r1s2w_c0.log
timeout 200 python scripts/prof_host.py c0 2>&1 | head -1 >> gpurun_out/r1s2w_c0.log
