cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for p in 0 30 60 100; do
  echo "L2PF=$p"; SVMB200_L2PF=$p timeout 300 python scripts/repeat_train.py c4 2 2>&1 | tail -2
done
SVMB200_L2PF=60 timeout 300 python scripts/repeat_train.py c2 2 2>&1 | tail -1
