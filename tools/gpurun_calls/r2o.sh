mkdir -p gpurun_out
timeout -s KILL 300 python tools/dbg_stream.py 256 8 32000 1024 > gpurun_out/r2o_tl_cfg2_fused.txt 2>&1
timeout -s KILL 600 python -m pytest tests/test_fused_step.py tests/test_gpu_parity.py -x -q > gpurun_out/r2o_tests.log 2>&1
tail -3 gpurun_out/r2o_tests.log
timeout -s KILL 300 python bench.py --config cfg2 --no-cpu-baseline --no-e2e > gpurun_out/r2o_bench_cfg2.json 2> gpurun_out/r2o_bench_cfg2.err
timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2o_bench_cfg3.json 2> gpurun_out/r2o_bench_cfg3.err
cat gpurun_out/r2o_tl_*.txt
for f in gpurun_out/r2o_bench_cfg2.json gpurun_out/r2o_bench_cfg3.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', d['ms_per_step']*1e3, d['select_verify_latency_us'], d['roofline']['frac'], d['roofline']['step_frac'])
"; done
timeout -s KILL 600 python -m pytest tests/test_greedy_gpu.py -x -q > gpurun_out/r2o_greedy_tests.log 2>&1
tail -3 gpurun_out/r2o_greedy_tests.log
timeout -s KILL 300 python bench.py --config cfg1 --no-cpu-baseline --no-e2e > gpurun_out/r2o_bench_cfg1.json 2> gpurun_out/r2o_bench_cfg1.err
python -c "
import json
d=json.loads(open('gpurun_out/r2o_bench_cfg1.json').read().strip().splitlines()[-1])
print('cfg1', d['ms_per_step']*1e3, d['select_verify_latency_us'], d['gpu_launches'])
"
