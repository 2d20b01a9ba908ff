timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 300 gpurun_out/bench_c4.err
timeout 1500 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -c 300 gpurun_out/bench_c5.err
for c in c4 c5; do python -c "
import json;l=json.load(open('gpurun_out/bench_$c.json'))
print('$c', 'value', round(l['value'],4), 'us/it', round(l['us_per_iteration'],2), 'iters', l['iterations'], 'frac', round(l['roofline']['frac'],3), 'traffic', l['roofline']['traffic'], 'e2e', round(l['e2e']['value'],4), 'cert_ms', round(l['train_breakdown_ms']['certify'],1), 'clk', l['clocks'])
"; done
