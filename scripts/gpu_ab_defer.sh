for rep in 1 2; do for v in base simple; do for d in 1 0; do
  if [ $v = base ]; then so=""; else so="build/ab_$v.so"; fi
  XMHD_SO=$so XMHD_PDEFER=$d timeout 120 python scripts/prof_leja.py 2048 48 2>&1 | grep fused | sed "s/^/$v defer=$d /" >> gpurun_out/r1s2r_ab.log
  XMHD_SO=$so XMHD_PDEFER=$d timeout 120 python scripts/prof_leja.py 4096 24 2>&1 | grep fused | sed "s/^/$v defer=$d /" >> gpurun_out/r1s2r_ab.log
done; done; done
