timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1s2b_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1s2b_pytest_gpu.log
for v in base pf3 pf4 pf3e2 base; do
  if [ $v = base ]; then so=""; else so="build/ab_$v.so"; fi
  echo "== $v" >> gpurun_out/r1s2b_ab.log
  XMHD_SO=$so timeout 120 python scripts/prof_leja.py 2048 48 >> gpurun_out/r1s2b_ab.log 2>&1
  XMHD_SO=$so timeout 120 python scripts/prof_leja.py 4096 24 >> gpurun_out/r1s2b_ab.log 2>&1
done
timeout 300 python scripts/prof_host.py c0 > gpurun_out/r1s2b_host_c0.log 2>&1
echo done
