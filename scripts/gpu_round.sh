timeout 600 python bench.py > gpurun_out/r1s2u_bench.json 2> gpurun_out/r1s2u_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r1s2u_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-exprb > gpurun_out/r1s2u_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel --launch-skip 2 -c 2 -o gpurun_out/r1s2u_leja python scripts/prof_leja.py 2048 3 > gpurun_out/r1s2u_ncu_full.log 2>&1
