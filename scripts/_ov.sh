cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "predict or ovr or closed or end_to_end or tight or tiny" 2>&1 | tail -2
timeout 300 python scripts/cert_probe.py c4 2>&1
timeout 300 python scripts/cert_probe.py c2 2>&1
