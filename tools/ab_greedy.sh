# A/B of two library builds on the greedy configs, interleaved, 3 rounds; usage: bash tools/ab_greedy.sh libA.so libB.so
mkdir -p gpurun_out
for r in 1 2 3; do for v in "$@"; do for c in cfg3g cfg1; do
  TETRIS_LIB_VARIANT=$v timeout -s KILL 300 python bench.py --config $c --steps 300 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/abg_$c.json 2>/dev/null
  python -c "import json;d=json.loads(open(\"gpurun_out/abg_$c.json\").read().strip().splitlines()[-1]);print(\"$v $c\",round(d[\"ms_per_step\"]*1000,2))"
done; done; done
