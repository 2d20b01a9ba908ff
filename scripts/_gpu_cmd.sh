export SVMB200_PROFILE=1
timeout 900 python scripts/prof_train.py c5:200000 300 2>&1 | tail -3
timeout 900 python scripts/prof_train.py c5 100 2>&1 | tail -3
unset SVMB200_PROFILE
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
