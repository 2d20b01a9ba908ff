timeout 2400 python bench.py --config c5 --steps 1 --warmup 3 --cpu-seconds 15 > gpurun_out/bench_c5.log 2>&1; echo rc=$?; tail -c 600 gpurun_out/bench_c5.log
