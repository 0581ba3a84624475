# A/B: cfg1 (greedy one launch) on the session's starting kernels (0383bcd) vs the final code
mkdir -p gpurun_out
for r in 1 2 3; do for v in libhead.so libtetris_b200.so; do
  TETRIS_LIB_VARIANT=$v timeout -s KILL 120 python bench.py --config cfg1 --steps 2000 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r2av_ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2av_ab.json').read().strip().splitlines()[-1]);print('$v cfg1',round(d['ms_per_step']*1000,2))"
done; done
