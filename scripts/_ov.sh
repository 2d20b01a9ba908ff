cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -q -x -m gpu 2>&1 | tail -2
timeout 60 python scripts/prof_train.py c2 0; timeout 60 python scripts/prof_train.py c4 8000; timeout 60 python scripts/prof_c3.py; timeout 100 python scripts/prof_train.py c5:400000 60
