timeout 600 python scripts/repeat_train.py c2 8
timeout 600 python scripts/repeat_train.py c4 4
