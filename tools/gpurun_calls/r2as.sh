# A/B: the sampler's per-request counter flush every 8 / 16 published chunks on large streams vs every 32 (HEAD), cfg3
mkdir -p gpurun_out
for r in 1 2 3; do for v in libhead.so libfl8.so libfl16.so; do
  for inp in probs logits; do
  TETRIS_LIB_VARIANT=$v timeout -s KILL 120 python bench.py --config cfg3 --input $inp --steps 500 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2as_ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2as_ab.json').read().strip().splitlines()[-1]);print('$v cfg3 $inp',round(d['ms_per_step']*1000,2))"
  done
done; done
