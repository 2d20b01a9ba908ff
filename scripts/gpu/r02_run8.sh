timeout 1200 python -m pytest tests/test_gpu_cv.py tests/test_gpu_golden.py -x -q -s 2>&1 | grep -v "^$" | tail -25
timeout 900 python -m pytest tests/test_gpu_paths.py -x -q 2>&1 | tail -4
