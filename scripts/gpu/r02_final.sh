timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_c4_final.json 2> gpurun_out/bench_c4_final.err; tail -c 300 gpurun_out/bench_c4_final.err
python -c "
import json;l=json.load(open('gpurun_out/bench_c4_final.json'))
print('c4', 'value', round(l['value'],4), 'us/it', round(l['us_per_iteration'],2), 'frac', round(l['roofline']['frac'],3), 'pass_only', round(l['roofline']['pass_only']['frac'],3), 'e2e', round(l['e2e']['value'],4), 'launches', l['gpu_launches'], 'clk', l['clocks'])
"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c4_launches_final.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-pass > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
