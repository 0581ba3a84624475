# A/B: the one-launch producer claims its next item after issuing the current copy (vs before it, HEAD)
mkdir -p gpurun_out
TETRIS_LIB_VARIANT=libcai.so timeout -s KILL 300 python -m pytest tests/test_fused_step.py -x -q 2>&1 | tail -1
for r in 1 2 3; do for v in libhead.so libcai.so; do
  for c in cfg2 cfg1; do
  TETRIS_LIB_VARIANT=$v timeout -s KILL 120 python bench.py --config $c --steps 2000 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r2az_ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2az_ab.json').read().strip().splitlines()[-1]);print('$v $c',round(d['ms_per_step']*1000,2))"
  done
done; done
