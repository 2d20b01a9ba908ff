timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 1200 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -c 400 gpurun_out/bench_c5.err
python -c "
import json;l=json.load(open('gpurun_out/bench_c5.json'))
print('c5', 'value', round(l['value'],3), 'us/it', round(l['us_per_iteration'],1), 'iters', l['iterations'], 'frac', round(l['roofline']['frac'],3), 'e2e', round(l['e2e']['value'],3), 'clk', l['clocks'])
"
