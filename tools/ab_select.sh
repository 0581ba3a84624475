# A/B of two builds of the library (TETRIS_LIB_VARIANT) on the step benches; usage: bash tools/ab_select.sh libA.so libtetris_b200.so
mkdir -p gpurun_out
for v in "$@"; do for c in cfg3 cfg1 cfg2; do
  TETRIS_LIB_VARIANT=$v timeout -s KILL 300 python bench.py --config $c --steps 1000 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}_$c.json 2>/dev/null
  python -c "import json;d=json.loads(open(\"gpurun_out/ab_${v}_$c.json\").read().strip().splitlines()[-1]);print(\"$v $c\",round(d[\"ms_per_step\"]*1000,2),{k:round(x,1) for k,x in d[\"stage_us\"].items()},round(d[\"roofline\"][\"frac\"],3))"
done; done
