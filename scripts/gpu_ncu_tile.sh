timeout 600 ncu --set full --clock-control none --import-source on -k regex:leja_tile_loop -c 1 -o gpurun_out/r1s2_tile128 python scripts/prof_tile.py 128 > gpurun_out/r1s2_ncu_tile.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:leja_tile_loop -c 1 -o gpurun_out/r1s2_tile512 python scripts/prof_tile.py 512 >> gpurun_out/r1s2_ncu_tile.log 2>&1
echo done
