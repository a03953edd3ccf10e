timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1s3d_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r1s3d_smoke.log
timeout 900 python bench.py > gpurun_out/r1s3d_bench.json 2> gpurun_out/r1s3d_bench.err; echo "bench rc=$?" >> gpurun_out/r1s3d_smoke.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1s3d_ref.json 2>> gpurun_out/r1s3d_bench.err
