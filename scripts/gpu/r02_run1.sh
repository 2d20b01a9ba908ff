set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_gpu_paths.py -x -q 2>&1 | tail -30 > gpurun_out/paths.log
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_paths.py 2>&1 | tail -30 > gpurun_out/gpu_all.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
tail -3 gpurun_out/paths.log gpurun_out/gpu_all.log; cat gpurun_out/bench_c4.json | head -c 3000
