timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu_all.log
SVMB200_PROFILE=1 timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_c3.log 2> gpurun_out/bench_c3.err; echo bench3_rc=$?; grep "batched OvR\|certify" gpurun_out/bench_c3.err | tail -3
SVMB200_PROFILE=1 timeout 600 python scripts/prof_train.py c5 3000 2>&1 | tail -4
