for v in base t3 t4; do
  if [ $v = base ]; then so=""; else so="build/ab_$v.so"; fi
  echo "== $v" >> gpurun_out/r1s2f_tile.log
  XMHD_SO=$so timeout 120 python scripts/prof_tile.py 128 512 >> gpurun_out/r1s2f_tile.log 2>&1
done
echo "== sliding loop" >> gpurun_out/r1s2f_tile.log
XMHD_TILE=0 timeout 120 python scripts/prof_tile.py 128 512 >> gpurun_out/r1s2f_tile.log 2>&1
echo "== per-term launches" >> gpurun_out/r1s2f_tile.log
XMHD_LOOP_MAX_CELLS=0 timeout 120 python scripts/prof_tile.py 128 512 >> gpurun_out/r1s2f_tile.log 2>&1
