timeout 900 python bench.py --impl reference > gpurun_out/ref_final.json 2> gpurun_out/ref_final.err; tail -c 300 gpurun_out/ref_final.err
python -c "
import json;l=json.load(open('gpurun_out/ref_final.json'))
print({k:l[k] for k in ('impl','value','unit','steps','warmup','ms_per_step')}, l['cpu_baseline'].get('sample'), l['config']['workload'])
"
