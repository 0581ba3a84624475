# A/B: segment sums published for short rows (descent re-reads one segment) vs HEAD
mkdir -p gpurun_out
timeout -s KILL 500 python -m pytest tests/test_gpu_parity.py tests/test_logits_gpu.py tests/test_fused_step.py -x -q > gpurun_out/r2an_tests.log 2>&1
tail -3 gpurun_out/r2an_tests.log
for r in 1 2 3; do for v in libhead.so libtetris_b200.so; do
  for c in cfg2 cfg3; do
  TETRIS_LIB_VARIANT=$v timeout -s KILL 120 python bench.py --config $c --steps 1000 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2an_ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2an_ab.json').read().strip().splitlines()[-1]);print('$v $c',round(d['ms_per_step']*1000,2))"
  done
  TETRIS_LIB_VARIANT=$v timeout -s KILL 120 python bench.py --input logits --steps 500 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2an_ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2an_ab.json').read().strip().splitlines()[-1]);print('$v cfg3 logits',round(d['ms_per_step']*1000,2))"
done; done
