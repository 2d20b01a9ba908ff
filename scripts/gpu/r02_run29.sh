SWEEP_CFG=c5 PROBE_N=500000 PASSES=10 timeout 300 python scripts/pass_probe.py 2>&1 | tail -1
SWEEP_CFG=c5 PROBE_N=500000 PASSES=10 timeout 900 ncu --set full --import-source on --clock-control none -k regex:smo_persistent -s 1 -c 1 -o gpurun_out/sell_c5 python scripts/pass_probe.py > gpurun_out/sell_ncu.log 2>&1; tail -2 gpurun_out/sell_ncu.log
SWEEP_CFG=c5 ITERS=3000 timeout 600 python scripts/train_probe.py 2>&1 | tail -1
SVMB200_CSR_STAGED=1 SWEEP_CFG=c5 ITERS=3000 timeout 600 python scripts/train_probe.py 2>&1 | tail -1
