mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_fused_step.py -x -q > gpurun_out/r2w_tests.log 2>&1
tail -5 gpurun_out/r2w_tests.log
for r in 1 2 3; do for v in libhead.so libtetris_b200.so; do for c in cfg3 cfg2; do
  TETRIS_LIB_VARIANT=$v timeout -s KILL 300 python bench.py --config $c --steps 1000 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2w_ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2w_ab.json').read().strip().splitlines()[-1]);print('$v $c',round(d['ms_per_step']*1000,2), round(d['roofline']['frac'],4))"
done; done; done
