mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_fused_step.py -x -q > gpurun_out/r2b_fused_tests.log 2>&1
tail -3 gpurun_out/r2b_fused_tests.log
timeout -s KILL 300 python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/r2b_bench_cfg2.json 2> gpurun_out/r2b_bench_cfg2.err
TETRIS_NO_FUSED=1 timeout -s KILL 300 python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/r2b_bench_cfg2_nofused.json 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_logits_gpu.py tests/test_policies.py tests/test_host_step.py -x -q > gpurun_out/r2b_tests.log 2>&1
tail -3 gpurun_out/r2b_tests.log
