mkdir -p gpurun_out
timeout -s KILL 400 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
for c in cfg1 cfg2 cfg3g cfg4; do
  timeout -s KILL 300 python bench.py --config $c > gpurun_out/r2f_bench_$c.json 2> gpurun_out/r2f_bench_$c.err
done
timeout -s KILL 300 python bench.py --input logits > gpurun_out/r2f_bench_logits.json 2> gpurun_out/r2f_bench_logits.err
for f in gpurun_out/r2f_bench*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
r=d.get('roofline') or {}; e=d.get('e2e') or {}
print('$f', round(d['ms_per_step']*1e3,2) if d.get('ms_per_step') else d.get('value'), r.get('frac'), r.get('step_frac'), e.get('ms_per_step'), d.get('clocks',{}).get('reasons'))
" || tail -3 ${f%.json}.err; done
