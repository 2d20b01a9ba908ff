timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ragged or csr" 2>&1 | tail -2
export SVMB200_CACHE=0 SWEEP_CFG=c5 ITERS=2000
timeout 600 python scripts/train_probe.py 2>&1 | tail -1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:smo_persistent -c 1 --csv --log-file gpurun_out/c5_dram.csv python scripts/train_probe.py > gpurun_out/c5_tp_ncu.log 2>&1; tail -1 gpurun_out/c5_tp_ncu.log; tail -3 gpurun_out/c5_dram.csv
