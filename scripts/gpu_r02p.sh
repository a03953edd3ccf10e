#!/bin/bash
# re-entry checkpoint: full GPU suite + smoke at HEAD, then the XB_P3EARLY A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02p_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02p_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02p_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02p_smoke.txt
V=paper_2108_13622_b200/_xmhd_b200_p3.so
for a in "2048 kh" "4096 kh" "2048 harris"; do
  echo "== $a"; timeout 300 python scripts/prof_leja_kinds.py $a 2>&1 | tail -1
  XMHD_SO=$V timeout 300 python scripts/prof_leja_kinds.py $a 2>&1 | tail -1
done
echo "== modes"; timeout 300 python scripts/prof_modes.py 2048 2>&1 | grep n=; XMHD_SO=$V timeout 300 python scripts/prof_modes.py 2048 2>&1 | grep n=
XMHD_SO=$V timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -m gpu -q -x > gpurun_out/r02p_pytest_p3.txt 2>&1; echo "pytest(p3) rc=$?"; tail -2 gpurun_out/r02p_pytest_p3.txt
timeout 600 python scripts/prof_timeline.py c4 3 > gpurun_out/r02p_timeline_c4.txt 2>&1; echo "timeline rc=$?"; tail -40 gpurun_out/r02p_timeline_c4.txt
