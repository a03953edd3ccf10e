#!/bin/bash
# adaptive runs over y-strips with real ranks (sharing the one GPU over gloo): counters against the one-rank run
for cfg in "3 3" "2 12"; do
echo "== config $cfg, 1 rank"; timeout 600 python scripts/run_config.py $cfg 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d.get('ranks'), d['accepted'], d['rejected'], d['rhs_evals'], d['phi_iterations'], d['t_reached'], d['checksum'][:12], round(d['wall_s'],2))"
for N in 2 3; do
echo "== config $cfg, $N ranks"; XMHD_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29517 scripts/run_config.py $cfg 2> gpurun_out/r03j_err.txt | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d.get('ranks'), d['accepted'], d['rejected'], d['rhs_evals'], d['phi_iterations'], d['t_reached'], d['checksum'][:12], round(d['wall_s'],2))" || tail -20 gpurun_out/r03j_err.txt
done
done
