#!/bin/bash
# r02: WS kernel diagnosis: timing of the three variants + one ncu capture
mkdir -p gpurun_out
for v in ws notma one; do
  case $v in
    ws) env="";;
    notma) env="XMHD_SO=paper_2108_13622_b200/_xmhd_b200_notma.so";;
    one) env="XMHD_WS=0";;
  esac
  echo "== $v"; env $env timeout 300 python scripts/prof_leja.py 2048 24 2>&1 | tail -2
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil_ws_kernel --launch-skip 2 -c 2 -o gpurun_out/r02f_ws python scripts/prof_leja.py 2048 3 > gpurun_out/r02f_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/r02f_ncu.log
