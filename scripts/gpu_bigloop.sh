echo "== per-term (default for 2048)" > gpurun_out/r1s2k_big.log
timeout 200 python scripts/prof_tile.py 2048 >> gpurun_out/r1s2k_big.log 2>&1
echo "== sliding loop" >> gpurun_out/r1s2k_big.log
XMHD_TILE=0 XMHD_LOOP_MAX_CELLS=67108864 timeout 200 python scripts/prof_tile.py 2048 >> gpurun_out/r1s2k_big.log 2>&1
echo "== tile loop" >> gpurun_out/r1s2k_big.log
XMHD_LOOP_MAX_CELLS=67108864 timeout 200 python scripts/prof_tile.py 2048 >> gpurun_out/r1s2k_big.log 2>&1
