export SWEEP_CFG=c5 PROBE_N=500000 PASSES=10
python scripts/pass_probe.py > gpurun_out/probe_c5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:smo_persistent -s 1 -c 1 -o gpurun_out/r02_pass_c5 python scripts/pass_probe.py > gpurun_out/ncu_c5.log 2>&1
cat gpurun_out/probe_c5_plain.log; tail -n 2 gpurun_out/ncu_c5.log
