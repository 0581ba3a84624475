mkdir -p gpurun_out
for w in 2 4 8; do
  timeout -s KILL 400 python bench.py --simulate-world $w --no-cpu-baseline --no-e2e > gpurun_out/r2ag_cfg3_w$w.json 2>/dev/null
done
for w in 4 8; do
  timeout -s KILL 400 python bench.py --config cfg5 --simulate-world $w --no-cpu-baseline --no-e2e > gpurun_out/r2ag_cfg5_w$w.json 2>/dev/null
done
for f in gpurun_out/r2ag_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', round(d['ms_per_step']*1e3,2), d['config']['workload'], d['config'].get('simulated_shard'), d['value'])
" || echo "$f failed"; done
