SVMB200_BENCH_N=100000 timeout 900 python bench.py --config c5 --steps 1 --warmup 3 --cpu-seconds 5 > gpurun_out/bench_c5_small.log 2>&1; echo rc=$?; tail -c 1500 gpurun_out/bench_c5_small.log
