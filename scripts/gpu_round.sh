set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r1s2_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1s2_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1s2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r1s2_smoke.log
timeout 600 python bench.py > gpurun_out/r1s2_bench.json 2> gpurun_out/r1s2_bench.err; echo "bench rc=$?"
timeout 300 python scripts/prof_leja.py 2048 20 > gpurun_out/r1s2_prof_leja.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r1s2_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-exprb > gpurun_out/r1s2_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel --launch-skip 2 -c 1 -o gpurun_out/r1s2_leja python scripts/prof_leja.py 2048 3 > gpurun_out/r1s2_ncu_full.log 2>&1
echo done
