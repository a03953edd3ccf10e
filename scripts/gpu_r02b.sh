#!/bin/bash
# r02 second pass: full GPU test suite, then the bench with the scale case
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/r02b_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_pytest.txt
tail -5 gpurun_out/r02b_pytest.txt
python bench.py --steps 5 --warmup 3 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02b_bench.err
python bench.py --gpus 2 --steps 1 --warmup 3 > gpurun_out/r02b_gpus2.out 2>&1; echo "gpus2 rc=$? (expect 2)"
