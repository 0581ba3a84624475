# A/B: the sampler's per-request counter flush every 1 / 2 / 4 published chunks on small streams (<= 2048 items) vs
# every 32 (HEAD)
mkdir -p gpurun_out
TETRIS_LIB_VARIANT=libflush1.so timeout -s KILL 300 python -m pytest tests/test_fused_step.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for r in 1 2; do for v in libhead.so libflush1.so libflush2.so libflush4.so; do
  for inp in probs logits; do
  TETRIS_LIB_VARIANT=$v timeout -s KILL 120 python bench.py --config cfg2 --input $inp --steps 1000 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2ar_ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2ar_ab.json').read().strip().splitlines()[-1]);print('$v cfg2 $inp',round(d['ms_per_step']*1000,2))"
  done
done; done
