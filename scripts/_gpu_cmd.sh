# end-of-round measurement refresh: GPU tests, bench lines (c2 headline, c3, c4), c2 launch list + ncu of the headline kernel
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu_all.log
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1; echo bench_rc=$?
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_c3.log 2>&1; echo bench3_rc=$?
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_c4.log 2>&1; echo bench4_rc=$?
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo benchref_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_c2.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_c3.log 2>&1; echo ncu2_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_decision_f16 -c 1 -o gpurun_out/dec_f16_c2 python scripts/predict_probe.py c2 > gpurun_out/ncu_dec_c2.log 2>&1; echo ncu3_rc=$?
