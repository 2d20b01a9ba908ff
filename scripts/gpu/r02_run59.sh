timeout 1800 python -m pytest tests/test_gpu_paths.py tests/test_gpu_golden.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 900 python bench.py --no-cpu > gpurun_out/bench_c4_ov.json 2> gpurun_out/bench_c4_ov.err; tail -c 200 gpurun_out/bench_c4_ov.err
python -c "
import json;l=json.load(open('gpurun_out/bench_c4_ov.json'))
print('c4', 'value', round(l['value'],4), 'us/it', round(l['us_per_iteration'],2), 'frac', round(l['roofline']['frac'],3), 'e2e', round(l['e2e']['value'],4), 'clk', l['clocks'])
"
