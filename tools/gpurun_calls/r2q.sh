# native NCCL sharded step (world 1, eager + graph), host-step tests, e2e copy issuance A/B
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_dist_gpu.py tests/test_host_step.py -x -q > gpurun_out/r2q_tests.log 2>&1
tail -3 gpurun_out/r2q_tests.log
timeout -s KILL 400 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/r2q_bench_threads.json 2> gpurun_out/r2q_bench_threads.err
TETRIS_SERIAL_COPIES=1 timeout -s KILL 400 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/r2q_bench_serial.json 2> gpurun_out/r2q_bench_serial.err
timeout -s KILL 400 python bench.py --no-cpu-baseline --steps 200 --nccl > gpurun_out/r2q_bench_nccl.json 2> gpurun_out/r2q_bench_nccl.err
timeout -s KILL 400 python bench.py --no-cpu-baseline --steps 200 --config cfg2 --nccl > gpurun_out/r2q_bench_cfg2_nccl.json 2> gpurun_out/r2q_bench_cfg2_nccl.err
for f in gpurun_out/r2q_bench_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', round(d['ms_per_step']*1e3,2), d['e2e'].get('ms_per_step') if d.get('e2e') else None, d['config']['parallelism'], d['config'].get('launch'))
" || tail -5 ${f%.json}.err; done
