# A/B: the plain / speculative producers claim after issuing the copy (vs before, HEAD) on cfg3 (+ logits), and the
# fused tests on the default build (the one-launch producer's claim-after-issue)
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_fused_step.py tests/test_logits_gpu.py -x -q 2>&1 | tail -1
TETRIS_LIB_VARIANT=libcai2.so timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for r in 1 2 3; do for v in libhead.so libcai2.so; do
  for inp in probs logits; do
  TETRIS_LIB_VARIANT=$v timeout -s KILL 120 python bench.py --config cfg3 --input $inp --steps 500 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2ba_ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2ba_ab.json').read().strip().splitlines()[-1]);print('$v cfg3 $inp',round(d['ms_per_step']*1000,2))"
  done
done; done
