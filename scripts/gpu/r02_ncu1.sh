python scripts/pass_probe.py > gpurun_out/probe_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:smo_persistent -s 1 -c 1 -o gpurun_out/r02_pass_c4 python scripts/pass_probe.py > gpurun_out/ncu1.log 2>&1
tail -3 gpurun_out/probe_plain.log gpurun_out/ncu1.log
