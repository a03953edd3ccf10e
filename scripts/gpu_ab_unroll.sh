for v in base un3 base un3; do
  if [ $v = base ]; then so=""; else so="build/ab_$v.so"; fi
  echo "== $v" >> gpurun_out/r1s2i_ab.log
  XMHD_SO=$so timeout 120 python scripts/prof_leja.py 2048 48 2>&1 | grep fused >> gpurun_out/r1s2i_ab.log
  XMHD_SO=$so timeout 120 python scripts/prof_leja.py 4096 24 2>&1 | grep fused >> gpurun_out/r1s2i_ab.log
done
XMHD_SO=build/ab_un3.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r1s2i_parity_un3.log 2>&1; echo "rc=$?" >> gpurun_out/r1s2i_parity_un3.log
echo done
