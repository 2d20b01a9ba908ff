SWEEP_CFG=c5 PROBE_N=500000 PASSES=10 timeout 300 python scripts/pass_probe.py 2>&1 | tail -1
SWEEP_CFG=c5 PROBE_N=500000 PASSES=10 timeout 900 ncu --set full --import-source on --clock-control none -k regex:smo_persistent -s 1 -c 1 -o gpurun_out/sell2_c5 python scripts/pass_probe.py > gpurun_out/sell2_ncu.log 2>&1; tail -1 gpurun_out/sell2_ncu.log
