cd $GRAFT_REPO_ROOT
for kv in "X=0" "SVMB200_OVERLAP=1" "SVMB200_XRING=0" "SVMB200_NO_DBUF=1" "SVMB200_NO_L2PERSIST=1"; do
  echo "$kv"; env $kv timeout 300 python scripts/repeat_train.py c4 2 2>&1 | tail -1 | cut -c1-110
done
