cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -2
python scripts/e2e_margins.py
python scripts/prof_train.py c2 0; python scripts/prof_train.py c4 8000; python scripts/prof_c3.py
