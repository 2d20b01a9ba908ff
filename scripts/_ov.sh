cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "partition or end_to_end or one_step" 2>&1 | tail -2
timeout 60 python scripts/prof_train.py c2 0; SVMB200_NO_FLAT=1 timeout 60 python scripts/prof_train.py c2 0; timeout 60 python scripts/prof_train.py c2 0
