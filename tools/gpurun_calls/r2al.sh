mkdir -p gpurun_out
TETRIS_LIB_VARIANT=libqint.so timeout -s KILL 400 python -m pytest tests/test_gpu_parity.py -x -q -k "adversarial or step or sampler" > gpurun_out/r2al_tests.log 2>&1
tail -2 gpurun_out/r2al_tests.log
for r in 1 2 3; do for v in libhead.so libqint.so; do
  TETRIS_LIB_VARIANT=$v timeout -s KILL 120 python bench.py --steps 1000 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2al_ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2al_ab.json').read().strip().splitlines()[-1]);print('$v cfg3',round(d['ms_per_step']*1000,2), round(d['roofline']['frac'],4))"
done; done
