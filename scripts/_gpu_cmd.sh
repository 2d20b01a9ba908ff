timeout 600 python scripts/prof_train.py c5 3000 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x -k "csr or CSR or c5 or kernel_rows" > gpurun_out/pytest_csr.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_csr.log
