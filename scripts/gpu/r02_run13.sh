timeout 900 python -m pytest tests/test_gpu_paths.py -x -q 2>&1 | tail -5
timeout 1500 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -c 400 gpurun_out/bench_c5.err; head -c 1200 gpurun_out/bench_c5.json
