# final validation (r2k): full GPU suite, smoke, default bench line, cfg2 / cfg1 / logits lines
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests/ -q -m gpu > gpurun_out/r2k_gpu_tests.log 2>&1
tail -2 gpurun_out/r2k_gpu_tests.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 600 python bench.py > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
for c in cfg2 cfg1; do timeout -s KILL 300 python bench.py --config $c > gpurun_out/r2k_bench_$c.json 2> gpurun_out/r2k_bench_$c.err; done
timeout -s KILL 300 python bench.py --input logits > gpurun_out/r2k_bench_logits.json 2> gpurun_out/r2k_bench_logits.err
