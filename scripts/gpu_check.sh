timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r1s3i_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r1s3i_pytest.log
for mb in 2 1; do echo "== minb $mb" >> gpurun_out/r1s3i_tile.log; XMHD_TILE_MINB=$mb timeout 200 python scripts/prof_tile.py 128 2>&1 | grep "n=" >> gpurun_out/r1s3i_tile.log; done
echo "== auto 512" >> gpurun_out/r1s3i_tile.log; timeout 200 python scripts/prof_tile.py 512 2>&1 | grep "n=" >> gpurun_out/r1s3i_tile.log
for i in 1 2; do for mb in 2 1; do XMHD_TILE_MINB=$mb timeout 200 python scripts/prof_host.py c0 2>&1 | head -1 | sed "s/^/minb=$mb /" >> gpurun_out/r1s3i_tile.log; done; done
