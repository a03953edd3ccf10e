#!/bin/bash
# A/B: XB_P3EARLY=1 variant (paper_2108_13622_b200/_xmhd_b200_p3.so) vs default
V=paper_2108_13622_b200/_xmhd_b200_p3.so
for a in "2048 kh" "4096 kh" "2048 harris"; do
  echo "== $a"; timeout 300 python scripts/prof_leja_kinds.py $a 2>&1 | tail -1
  XMHD_SO=$V timeout 300 python scripts/prof_leja_kinds.py $a 2>&1 | tail -1
done
echo "== modes"; timeout 300 python scripts/prof_modes.py 2048 2>&1 | grep n=; XMHD_SO=$V timeout 300 python scripts/prof_modes.py 2048 2>&1 | grep n=
XMHD_SO=$V timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02o_pytest.txt 2>&1; echo "pytest(p3) rc=$?"; tail -2 gpurun_out/r02o_pytest.txt
