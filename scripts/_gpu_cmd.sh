timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_all.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu_all.log
timeout 600 python scripts/predict_probe.py c2 2>&1 | tail -1
