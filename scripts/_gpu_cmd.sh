timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu_all.log
timeout 600 python scripts/repeat_train.py c2 3 2>&1 | tail -1
timeout 600 python scripts/repeat_train.py c3 3 2>&1 | tail -1
timeout 600 python scripts/e2e_margins.py > gpurun_out/margins.log 2>&1; tail -3 gpurun_out/margins.log
