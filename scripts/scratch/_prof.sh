cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SVMB200_PROFILE_BUILD=1 python -c "from paper_1706_05544_b200 import _build; _build.build(force=True)" > gpurun_out/profbuild.log 2>&1; echo "build rc=$?"
for c in c4 c2; do
SVMB200_PROFILE=1 timeout 300 python scripts/prof_train.py $c 0 2>&1 | grep -E "svmb200|iters" | tail -4
done
