# A/B of two library builds on the latency-bound configs, interleaved, 3 rounds: bash tools/ab_small.sh libA.so libB.so
mkdir -p gpurun_out
for r in 1 2 3; do for v in "$@"; do for c in cfg1 cfg2 cfg3; do
  TETRIS_LIB_VARIANT=$v timeout -s KILL 300 python bench.py --config $c --steps 1000 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/abs_$c.json 2>/dev/null
  python -c "import json;d=json.loads(open(\"gpurun_out/abs_$c.json\").read().strip().splitlines()[-1]);print(\"$v $c\",round(d[\"ms_per_step\"]*1000,2))"
done; done; done
