#!/bin/bash
# final_pair (embedded pair of a step in one pass): full GPU suite, config 3 / 4 steps
mkdir -p gpurun_out
T=r03a
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.txt
for fp in 1 0; do
XMHD_FINAL_PAIR=$fp timeout 600 python scripts/run_config.py 4 10 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c4 final_pair=$fp', d['accepted'], d['rhs_evals'], d['phi_iterations'], round(d['wall_s_per_step'],4), 'after first', round(d['wall_s_per_step_after_first'],4), d['checksum'][:12])"
XMHD_FINAL_PAIR=$fp timeout 600 python scripts/run_config.py 3 20 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c3 final_pair=$fp', d['accepted'], d['rhs_evals'], d['phi_iterations'], round(d['wall_s_per_step'],4), 'after first', round(d['wall_s_per_step_after_first'],4), d['checksum'][:12])"
done
