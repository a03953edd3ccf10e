#!/bin/bash
# A/B of two library builds on one box: usage gpu_ab.sh <variant.so> [more prof args]
V=$1
for rep in 1 2; do
for a in "2048 kh" "4096 kh" "2048 harris"; do
  echo "== $a (default, then $V)"; timeout 300 python scripts/prof_leja_kinds.py $a 2>&1 | tail -1 | sed 's/plan {[^}]*}//'
  XMHD_SO=$V timeout 300 python scripts/prof_leja_kinds.py $a 2>&1 | tail -1 | sed 's/plan {[^}]*}//'
done
done
echo "== modes"; timeout 300 python scripts/prof_modes.py 2048 2>&1 | grep n=; XMHD_SO=$V timeout 300 python scripts/prof_modes.py 2048 2>&1 | grep n=
