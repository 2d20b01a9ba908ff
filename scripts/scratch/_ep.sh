cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for c in c2 c4; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
  python -c "
import json; j=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); print(j['value'], j['iterations'], j['us_per_iteration'], j.get('exchange',{}).get('us_per_iteration'), j['roofline']['frac'], j['train_breakdown_ms']['per_step_train_ms'])"
done
