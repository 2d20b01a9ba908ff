cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
SVMB200_PROFILE=1 timeout 300 python scripts/cert_probe.py c4 2>&1 | grep -v "phases\|worker"
SVMB200_PROFILE=1 timeout 300 python scripts/cert_probe.py c2 2>&1 | grep -v "phases\|worker"
