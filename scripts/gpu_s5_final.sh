# session-5 closing pass: GPU suite, smoke, default bench, reference arm, launch list.
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s5f_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s5f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s5f_smoke.log
timeout 900 python bench.py > gpurun_out/s5f_bench.json 2> gpurun_out/s5f_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s5f_ref.json 2>> gpurun_out/s5f_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/s5f_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-exprb > gpurun_out/s5f_ncu_launch.log 2>&1
