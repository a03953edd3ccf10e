#!/bin/bash
# several variant builds against the default on one box (per-kind term times)
for rep in 1 2; do
for a in "2048 kh" "4096 kh"; do
  echo "== $a default"; timeout 300 python scripts/prof_leja_kinds.py $a 2>&1 | tail -1 | sed 's/plan {[^}]*}//'
  for v in "$@"; do echo -n "$v: "; XMHD_SO=paper_2108_13622_b200/_xmhd_b200_$v.so timeout 300 python scripts/prof_leja_kinds.py $a 2>&1 | tail -1 | sed 's/plan {[^}]*}//'; done
done
done
