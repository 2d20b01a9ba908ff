set -x
timeout 1500 python -m pytest tests/test_gpu_golden.py -x -q -s 2>&1 | tail -30 > gpurun_out/golden.log
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_golden.py 2>&1 | tail -30 > gpurun_out/gpu_all.log
tail -3 gpurun_out/golden.log gpurun_out/gpu_all.log
