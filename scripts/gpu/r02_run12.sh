timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
tail -c 600 gpurun_out/bench_c4.err
python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-pass > gpurun_out/ll_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_c4_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-pass > gpurun_out/ncu_ll.log 2>&1
python scripts/train_probe.py > gpurun_out/tp_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:smo_persistent -c 1 -o gpurun_out/r02_c4_persistent python scripts/train_probe.py > gpurun_out/ncu_tp.log 2>&1
tail -2 gpurun_out/tp_plain.log gpurun_out/ncu_tp.log gpurun_out/ncu_ll.log
