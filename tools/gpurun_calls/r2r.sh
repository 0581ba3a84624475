# staged host steps through the gather kernel: tests + e2e lines (fp32, logits, greedy cfg1)
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_host_step.py tests/test_logits_gpu.py tests/test_dist_gpu.py -x -q > gpurun_out/r2r_tests.log 2>&1
tail -3 gpurun_out/r2r_tests.log
timeout -s KILL 400 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/r2r_bench.json 2> gpurun_out/r2r_bench.err
timeout -s KILL 400 python bench.py --no-cpu-baseline --steps 200 --input logits > gpurun_out/r2r_bench_logits.json 2> gpurun_out/r2r_bench_logits.err
timeout -s KILL 400 python bench.py --no-cpu-baseline --steps 200 --config cfg3g > gpurun_out/r2r_bench_cfg3g.json 2> gpurun_out/r2r_bench_cfg3g.err
timeout -s KILL 400 python bench.py --no-cpu-baseline --steps 200 --nccl > gpurun_out/r2r_bench_nccl.json 2> gpurun_out/r2r_bench_nccl.err
for f in gpurun_out/r2r_bench*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', round(d['ms_per_step']*1e3,2), d['e2e'].get('ms_per_step') if d.get('e2e') else None, d['config']['parallelism'], d['config'].get('launch'))
" || tail -5 ${f%.json}.err; done
