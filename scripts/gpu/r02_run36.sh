timeout 900 python -m pytest tests/test_gpu_paths.py -q -x -k "increment or process" -s 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_cv.py -q -x 2>&1 | tail -2
SVMB200_PROFILE=1 timeout 900 python scripts/c5_train_once.py 2>&1 | grep -v "loop\|worker" | tail -5 || true
