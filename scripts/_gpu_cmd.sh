timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu_all.log
SVMB200_PROFILE=1 timeout 600 python scripts/repeat_train.py c3 3 2>&1 | grep "run\|certify:" | tail -4
