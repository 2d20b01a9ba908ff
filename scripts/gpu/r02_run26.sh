timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 300 gpurun_out/bench_c4.err
python -c "
import json;l=json.load(open('gpurun_out/bench_c4.json'))
print('c4', 'value', round(l['value'],4), 'us/it', round(l['us_per_iteration'],2), 'iters', l['iterations'], 'frac', round(l['roofline']['frac'],3), 'pass_only', round(l['roofline']['pass_only']['frac'],3), 'e2e', round(l['e2e']['value'],4), 'cpu', l['cpu_baseline'].get('value'), 'exch', l['exchange']['p50_us'], l['exchange']['p99_us'], 'clk', l['clocks'])
"
