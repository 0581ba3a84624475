mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_golden_scale.py tests/test_dist_gpu.py tests/test_dropin.py -x -q > gpurun_out/r2ac_tests.log 2>&1
tail -3 gpurun_out/r2ac_tests.log
for r in 1 2; do for v in libhead.so libtetris_b200.so; do
  TETRIS_LIB_VARIANT=$v timeout -s KILL 300 python bench.py --config cfg4 --steps 500 --warmup 5 > gpurun_out/r2ac_ab.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/r2ac_ab.json').read().strip().splitlines()[-1])
print('$v cfg4', {c: round(v['us_per_select'],2) for c, v in d['sweep'].items()})"
done; done
for c in 4096 8192 32768; do timeout -s KILL 120 python tools/dbg_gselect.py 4096 16 $c; done
