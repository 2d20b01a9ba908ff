cd $GRAFT_REPO_ROOT
for nb in 148 128 112 100; do echo "NBLK=$nb"; SVMB200_NBLK=$nb python scripts/prof_train.py c2 0; done
