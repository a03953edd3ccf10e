# One round of GPU evidence (run under gpurun from the repo root):
# parity suite, smoke, the default bench line, the ncu launch list of one
# bench step and a full ncu capture of two consecutive fused Leja terms.
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-exprb > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel --launch-skip 2 -c 2 -o gpurun_out/leja python scripts/prof_leja.py 2048 3 > gpurun_out/ncu_full.log 2>&1
