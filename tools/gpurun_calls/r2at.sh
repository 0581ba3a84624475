# A/B: logits form of the one-launch step: scans by the consumers of the first CTA to finish its stream vs the scanner
# warp (HEAD)
mkdir -p gpurun_out
timeout -s KILL 500 python -m pytest tests/test_gpu_parity.py tests/test_logits_gpu.py tests/test_fused_step.py -x -q > gpurun_out/r2at_tests.log 2>&1
tail -3 gpurun_out/r2at_tests.log
for r in 1 2 3; do for v in libhead.so libtetris_b200.so; do
  for inp in probs logits; do
  TETRIS_LIB_VARIANT=$v timeout -s KILL 120 python bench.py --config cfg2 --input $inp --steps 1000 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2at_ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2at_ab.json').read().strip().splitlines()[-1]);print('$v cfg2 $inp',round(d['ms_per_step']*1000,2))"
  done
done; done
timeout -s KILL 300 python tools/dbg_stream.py 256 8 32000 1024 2>&1 | head -16
