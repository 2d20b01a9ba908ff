cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py --no-cpu > gpurun_out/b_c2.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/b_c2.json').read().strip().splitlines()[-1]); print('c2', round(d['value'],4), d['us_per_iteration'], d['train_breakdown_ms'], round(d['predict_rows_per_s']), d['roofline']['frac'])"
timeout 900 python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/b_c4.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/b_c4.json').read().strip().splitlines()[-1]); print('c4', round(d['value'],4), d['us_per_iteration'], d['train_breakdown_ms'], round(d['predict_rows_per_s']), d['roofline']['frac'])"
