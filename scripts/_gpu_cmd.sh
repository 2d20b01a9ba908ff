# round-1 measurement refresh (after the batched OvR / d > 128 decision / CSR mask work)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu_all.log
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; echo bench_rc=$?
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_c3.log 2>&1; echo bench3_rc=$?
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_c4.log 2>&1; echo bench4_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_c3.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ovr_pass -s 20 -c 1 -o gpurun_out/ovr_pass_r01 python scripts/prof_ovr.py 32 > gpurun_out/ncu_ovr.log 2>&1; echo ncu2_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_decision_f16 -s 1 -c 1 -o gpurun_out/dec_f16_r01 python scripts/prof_cert.py > gpurun_out/ncu_dec.log 2>&1; echo ncu3_rc=$?
