for c in c2 c3 c5; do
  timeout 1500 python bench.py --config $c > gpurun_out/bench_${c}_final.json 2> gpurun_out/bench_${c}_final.err
  python -c "
import json;l=json.load(open('gpurun_out/bench_${c}_final.json'))
r=l['roofline']
print('$c', round(l['value'],4), l.get('iterations'), round(l.get('us_per_iteration') or 0,2), round(r['frac'],3), r['unit'], round(l['predict_rows_per_s']/1e6,2), l['certified'], l['clocks']['reasons'], 'e2e', round(l['e2e']['value'],4) if l.get('e2e') else None)
" || tail -c 300 gpurun_out/bench_${c}_final.err
done
