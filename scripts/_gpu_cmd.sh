timeout 600 python bench.py > gpurun_out/bench2.log 2>&1; echo bench_rc=$?; tail -c 2500 gpurun_out/bench2.log
timeout 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo ncu1_rc=$?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:smo_persistent -c 1 -o gpurun_out/smo_c2_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?; tail -2 gpurun_out/ncu_full.log
