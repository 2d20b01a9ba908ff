timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -s > gpurun_out/pytest_full.log 2>&1; echo full_rc=$?; tail -5 gpurun_out/pytest_full.log
timeout 300 python scripts/probe.py c4 > gpurun_out/probe_c4.log 2>&1; tail -4 gpurun_out/probe_c4.log
