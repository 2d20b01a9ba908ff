timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 300 gpurun_out/bench_c4.err
timeout 900 python bench.py --config c2 --steps 3 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -c 300 gpurun_out/bench_c2.err
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 300 gpurun_out/bench_c3.err
for c in c4 c2 c3; do python -c "
import json;l=json.load(open('gpurun_out/bench_$c.json'))
print('$c', 'value', round(l['value'],4), 'us/it', round(l['us_per_iteration'],2), 'iters', l['iterations'], 'frac', round(l['roofline']['frac'],3), 'pass_only', (round(l['roofline'].get('pass_only',{}).get('frac',0),3)), 'e2e', round(l['e2e']['value'],4), 'pred', round(l['predict_rows_per_s']/1e6,2), 'cpu', l['cpu_baseline'].get('value'), 'clk', l['clocks'])
"; done
