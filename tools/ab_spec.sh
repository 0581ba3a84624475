# A/B of the speculative sampler (default) against the plain one (TETRIS_NO_SPEC=1), interleaved, 3 rounds.
mkdir -p gpurun_out
for r in 1 2 3; do for v in 0 1; do for c in cfg3 cfg2; do
  TETRIS_NO_SPEC=$v timeout -s KILL 300 python bench.py --config $c --steps 1000 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/abs_$v_$c.json 2>/dev/null
  python -c "import json;d=json.loads(open(\"gpurun_out/abs_$v_$c.json\").read().strip().splitlines()[-1]);print(\"nospec=$v $c\",round(d[\"ms_per_step\"]*1000,2))"
done; done; done
