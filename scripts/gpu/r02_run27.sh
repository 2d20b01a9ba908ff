export ITERS=100000
timeout 300 python scripts/train_probe.py > gpurun_out/tp_full.log 2>&1; cat gpurun_out/tp_full.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:smo_persistent -c 1 --csv --log-file gpurun_out/c4_full_dram.csv python scripts/train_probe.py > gpurun_out/tp_ncu.log 2>&1; tail -3 gpurun_out/tp_ncu.log; cat gpurun_out/c4_full_dram.csv | tail -4
timeout 600 python -m pytest tests/test_gpu_paths.py -q -k process 2>&1 | tail -3
