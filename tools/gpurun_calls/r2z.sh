mkdir -p gpurun_out
for r in 1 2 3; do for v in libbase.so libs2.so; do for c in cfg2 cfg3; do
  TETRIS_LIB_VARIANT=$v timeout -s KILL 300 python bench.py --config $c --steps 1000 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2z_ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2z_ab.json').read().strip().splitlines()[-1]);print('$v $c',round(d['ms_per_step']*1000,2), round(d['roofline']['frac'],4))"
done; done; done
