timeout 300 python scripts/prof_train.py c2 0 2>&1 | tail -1
timeout 600 python scripts/prof_train.py c4 300 > gpurun_out/c4_300_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:smo_persistent -c 1 -o gpurun_out/smo_c4_v2 python scripts/prof_train.py c4 300 > gpurun_out/ncu_c4.log 2>&1; echo ncu_rc=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
