# A/B: the one-launch greedy producer's phase-B claim after the copy (vs before, HEAD), cfg1
mkdir -p gpurun_out
TETRIS_LIB_VARIANT=libgca.so timeout -s KILL 300 python -m pytest tests/test_greedy_gpu.py tests/test_fused_step.py -x -q 2>&1 | tail -1
for r in 1 2 3; do for v in libhead.so libgca.so; do
  TETRIS_LIB_VARIANT=$v timeout -s KILL 120 python bench.py --config cfg1 --steps 2000 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r2bb_ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2bb_ab.json').read().strip().splitlines()[-1]);print('$v cfg1',round(d['ms_per_step']*1000,2))"
done; done
