cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 60 python scripts/prof_train.py c2 0; timeout 60 python scripts/prof_train.py c4 8000; timeout 60 python scripts/prof_c3.py
