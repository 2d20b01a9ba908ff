timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ovr" > gpurun_out/pytest_ovr.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_ovr.log
SVMB200_PROFILE=1 timeout 300 python scripts/prof_ovr.py 64 2>&1 | grep -v "^\[svmb200\] certify"
timeout 600 python scripts/repeat_train.py c3 3 2>&1 | tail -1
