#!/bin/bash
# A/B: 3-slot FX/FY rings (70 KB) with 2 or 3 CTAs per SM (168 registers) vs the default build
mkdir -p gpurun_out
T=r03b
for V in build/ab_ring3m3.so build/ab_ring3.so; do
  echo "== parity $V"; XMHD_SO=$V timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
done
for rep in 1 2; do
for a in "2048 kh" "4096 kh" "2048 harris"; do
  echo "== $a default"; timeout 300 python scripts/prof_leja_kinds.py $a 2>&1 | tail -1 | sed 's/plan {[^}]*}//'
  for V in build/ab_ring3m3.so build/ab_ring3.so; do
  echo "   $V"; XMHD_SO=$V timeout 300 python scripts/prof_leja_kinds.py $a 2>&1 | tail -1 | sed 's/plan {[^}]*}//'
  done
done
done
echo "== modes"; timeout 300 python scripts/prof_modes.py 2048 2>&1 | grep n=
for V in build/ab_ring3m3.so build/ab_ring3.so; do XMHD_SO=$V timeout 300 python scripts/prof_modes.py 2048 2>&1 | grep n=; done
