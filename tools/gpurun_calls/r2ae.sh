mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_fused_step.py tests/test_greedy_gpu.py tests/test_host_step.py -x -q > gpurun_out/r2ae_tests.log 2>&1
tail -3 gpurun_out/r2ae_tests.log
for r in 1 2 3; do for v in libhead.so libtetris_b200.so; do
  TETRIS_LIB_VARIANT=$v timeout -s KILL 300 python bench.py --config cfg1 --steps 2000 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2ae_ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2ae_ab.json').read().strip().splitlines()[-1]);print('$v cfg1',round(d['ms_per_step']*1000,2), d['select_verify_latency_us'])"
done; done
timeout -s KILL 300 python tools/dbg_graph_greedy.py 16 5 32000 48
