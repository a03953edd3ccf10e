timeout 300 python scripts/prof_host.py c0 > gpurun_out/r1s2_host_c0.log 2>&1
timeout 300 python scripts/prof_host.py c2 1.0 > gpurun_out/r1s2_host_c2.log 2>&1
for n in 128 512; do timeout 120 python scripts/prof_leja.py $n 200 >> gpurun_out/r1s2_small_leja.log 2>&1; done
timeout 300 python scripts/prof_sweep.py > gpurun_out/r1s2_sweep.log 2>&1
timeout 120 python scripts/pcie_probe.py > gpurun_out/r1s2_pcie.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r1s2_c0_launches.csv python scripts/prof_host.py c0 0.1 > /dev/null 2>&1
echo done
