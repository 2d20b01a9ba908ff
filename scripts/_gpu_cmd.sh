export SVMB200_PROFILE=1
timeout 300 python scripts/probe.py c1 c2 > gpurun_out/probe5.log 2>&1; echo probe_rc=$?
grep -v "^\[svmb200\]" gpurun_out/probe5.log | tail; grep "^\[svmb200\]" gpurun_out/probe5.log | tail -4
unset SVMB200_PROFILE
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -25 gpurun_out/pytest_gpu.log
