timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r1s2g_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1s2g_pytest.log
timeout 120 python scripts/prof_tile.py 128 512 > gpurun_out/r1s2g_tile.log 2>&1
timeout 200 python scripts/prof_host.py c0 > gpurun_out/r1s2g_host_c0.log 2>&1
timeout 600 python scripts/run_config.py 2 > gpurun_out/r1s2g_c2.log 2>&1
echo done
timeout 300 python scripts/run_config.py 0 > gpurun_out/r1s2g_c0.log 2>&1
