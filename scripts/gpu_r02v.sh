#!/bin/bash
mkdir -p gpurun_out
show() { python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['accepted'], d['rhs_evals'], d['phi_iterations'], round(d['wall_s_per_step'],4), 'after first', round(d['wall_s_per_step_after_first'],4), d['step_wall_ms'][:12], d['checksum'][:12])"; }
for cfg in "XMHD_ADAPTIVE=0 XMHD_SPEC_TABLES=0" "XMHD_ADAPTIVE=1 XMHD_SPEC_TABLES=0" "XMHD_ADAPTIVE=1 XMHD_SPEC_TABLES=1" "XMHD_ADAPTIVE=0 XMHD_SPEC_TABLES=0 XMHD_FUSE_STAGES=0 XMHD_ZERO_COPY=0"; do
  echo "== $cfg"
  env $cfg timeout 600 python scripts/run_config.py 4 10 2>&1 | tail -1 | show
  env $cfg timeout 600 python scripts/run_config.py 3 20 2>&1 | tail -1 | show
done
