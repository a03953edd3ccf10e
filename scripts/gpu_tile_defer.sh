for d in 1 0; do echo "== defer $d" >> gpurun_out/r1s2v_tile.log; XMHD_PDEFER=$d timeout 200 python scripts/prof_tile.py 128 512 >> gpurun_out/r1s2v_tile.log 2>&1; done
timeout 200 python scripts/prof_host.py c0 2>&1 | head -1 > gpurun_out/r1s2v_c0.log
XMHD_PDEFER=0 timeout 200 python scripts/prof_host.py c0 2>&1 | head -1 >> gpurun_out/r1s2v_c0.log
