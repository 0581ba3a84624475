# round-2 re-entry check: full GPU suite, default bench, per-config lines, launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2p_smi.txt 2>&1
timeout -s KILL 1500 python -m pytest tests/ -x -q -m gpu > gpurun_out/r2p_gpu_tests.log 2>&1
tail -3 gpurun_out/r2p_gpu_tests.log
timeout -s KILL 400 python bench.py > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err
tail -c 3000 gpurun_out/r2p_bench.json
for c in cfg1 cfg2 cfg4; do
  timeout -s KILL 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2p_bench_$c.json 2> gpurun_out/r2p_bench_$c.err
done
timeout -s KILL 400 python bench.py --impl reference > gpurun_out/r2p_ref.json 2> gpurun_out/r2p_ref.err
tail -c 1500 gpurun_out/r2p_ref.json
