# final check of the final code (r2i): full GPU suite, smoke, the default bench line and the cfg2 / logits lines
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests/ -q -m gpu > gpurun_out/r2i_gpu_tests.log 2>&1
tail -2 gpurun_out/r2i_gpu_tests.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 600 python bench.py > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err
timeout -s KILL 300 python bench.py --config cfg2 > gpurun_out/r2i_bench_cfg2.json 2> gpurun_out/r2i_bench_cfg2.err
timeout -s KILL 300 python bench.py --config cfg1 > gpurun_out/r2i_bench_cfg1.json 2> gpurun_out/r2i_bench_cfg1.err
timeout -s KILL 300 python bench.py --input logits > gpurun_out/r2i_bench_logits.json 2> gpurun_out/r2i_bench_logits.err
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2i_ref_arm.json 2> gpurun_out/r2i_ref_arm.err
tail -c 400 gpurun_out/r2i_ref_arm.json
