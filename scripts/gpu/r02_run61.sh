timeout 1800 python -m pytest tests/test_gpu_paths.py -q -x -k "cache" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_c4_r2final.json 2> gpurun_out/bench_c4_r2final.err; tail -c 200 gpurun_out/bench_c4_r2final.err
python -c "
import json;l=json.load(open('gpurun_out/bench_c4_r2final.json'))
print('c4', 'value', round(l['value'],4), 'us/it', round(l['us_per_iteration'],2), 'frac', round(l['roofline']['frac'],3), 'pass', round(l['roofline']['pass_only']['frac'],3), 'cachep', l['roofline']['cache_passes'], 'e2e', round(l['e2e']['value'],4), 'clk', l['clocks'])
"
