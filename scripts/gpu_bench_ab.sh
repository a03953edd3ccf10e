for v in base sw64 sw64pf3; do
  if [ $v = base ]; then so=""; else so="build/ab_$v.so"; fi
  echo "== $v" >> gpurun_out/r1s2h_ab.log
  XMHD_SO=$so timeout 120 python scripts/prof_leja.py 2048 48 2>&1 | grep fused >> gpurun_out/r1s2h_ab.log
  XMHD_SO=$so timeout 120 python scripts/prof_leja.py 4096 24 2>&1 | grep fused >> gpurun_out/r1s2h_ab.log
done
timeout 600 python bench.py > gpurun_out/r1s2h_bench.json 2> gpurun_out/r1s2h_bench.err
echo done
