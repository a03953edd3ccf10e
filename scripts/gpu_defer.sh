timeout 600 python -m pytest tests/test_gpu_async.py -q -x > gpurun_out/r1s2t_async.log 2>&1; echo "rc=$?" >> gpurun_out/r1s2t_async.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r1s2t_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1s2t_pytest.log
for rep in 1 2; do for v in base simple; do
  if [ $v = base ]; then so=""; else so="build/ab_$v.so"; fi
  XMHD_SO=$so timeout 120 python scripts/prof_leja.py 2048 48 2>&1 | grep fused | sed "s/^/$v /" >> gpurun_out/r1s2t_ab.log
  XMHD_SO=$so timeout 120 python scripts/prof_leja.py 4096 24 2>&1 | grep fused | sed "s/^/$v /" >> gpurun_out/r1s2t_ab.log
done; done
timeout 300 python scripts/prof_sweep.py > gpurun_out/r1s2t_sweep.log 2>&1
