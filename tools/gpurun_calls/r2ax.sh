# final validation of the final code: full GPU suite, smoke, default bench line, the one-launch configs
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests/ -q -m gpu > gpurun_out/r2j_gpu_tests.log 2>&1
tail -2 gpurun_out/r2j_gpu_tests.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 600 python bench.py > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err
timeout -s KILL 300 python bench.py --config cfg2 > gpurun_out/r2j_bench_cfg2.json 2> gpurun_out/r2j_bench_cfg2.err
timeout -s KILL 300 python bench.py --config cfg1 > gpurun_out/r2j_bench_cfg1.json 2> gpurun_out/r2j_bench_cfg1.err
timeout -s KILL 300 python tools/sanitize.py > gpurun_out/r2j_sanitize_plain.txt 2>&1; tail -1 gpurun_out/r2j_sanitize_plain.txt
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py > gpurun_out/r2j_memcheck.txt 2>&1; tail -1 gpurun_out/r2j_memcheck.txt
