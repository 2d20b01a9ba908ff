cd $GRAFT_REPO_ROOT
SVMB200_PROFILE=1 timeout 600 python bench.py --config c3 --steps 4 --warmup 2 --no-cpu --no-e2e 2>gpurun_out/c3err.log | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['iterations'], d['train_breakdown_ms'])"
grep "certify:" gpurun_out/c3err.log | awk '{print $13}' | tr '\n' ' '; echo
grep "batched" gpurun_out/c3err.log
