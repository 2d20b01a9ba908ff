# round-1 measurement pass: GPU tests, bench lines (c2 headline, c4, c3), launch list, ncu full captures
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu_all.log
timeout 600 python bench.py > gpurun_out/bench_r01.log 2>&1; echo bench_rc=$?
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_r01_c4.log 2>&1; echo bench4_rc=$?
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_r01_c3.log 2>&1; echo bench3_rc=$?
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_r01_ref.log 2>&1; echo benchref_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_r01.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo ncu1_rc=$?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:smo_persistent -c 1 -o gpurun_out/smo_c2_r01 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:smo_persistent -c 1 -o gpurun_out/smo_c3_r01 python scripts/prof_c3.py > gpurun_out/ncu_full_c3.log 2>&1; echo ncu3_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_decision_tcp -s 2 -c 1 -o gpurun_out/dec_c2_r01 python scripts/predict_probe.py c2 > gpurun_out/ncu_dec.log 2>&1; echo ncu4_rc=$?
