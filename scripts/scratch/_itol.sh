cd $GRAFT_REPO_ROOT
for x in 0.1 0.3 1.0; do
  echo "inner_tol = $x tol"
  SVMB200_INNER_TOL_X=$x timeout 300 python scripts/repeat_train.py c4 2 2>&1 | tail -1
  SVMB200_INNER_TOL_X=$x timeout 300 python scripts/repeat_train.py c2 2 2>&1 | tail -1
done
