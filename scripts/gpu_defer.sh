timeout 600 python -m pytest tests/test_gpu_async.py -q -x > gpurun_out/r1s2q_async.log 2>&1; echo "rc=$?" >> gpurun_out/r1s2q_async.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r1s2q_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1s2q_pytest.log
for d in 1 0 1 0; do XMHD_PDEFER=$d timeout 120 python scripts/prof_leja.py 2048 48 2>&1 | grep fused | sed "s/^/defer=$d /" >> gpurun_out/r1s2q_defer.log; XMHD_PDEFER=$d timeout 120 python scripts/prof_leja.py 4096 24 2>&1 | grep fused | sed "s/^/defer=$d /" >> gpurun_out/r1s2q_defer.log; done
timeout 300 python scripts/prof_sweep.py > gpurun_out/r1s2q_sweep.log 2>&1
