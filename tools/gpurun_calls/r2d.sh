mkdir -p gpurun_out
timeout -s KILL 300 python tools/dbg_stream.py 256 8 32000 1024 > gpurun_out/r2d_tl_cfg2_fused.txt 2>&1
TETRIS_NO_FUSED=1 timeout -s KILL 300 python tools/dbg_stream.py 256 8 32000 1024 > gpurun_out/r2d_tl_cfg2_plain.txt 2>&1
timeout -s KILL 300 python tools/dbg_stream.py 1024 16 128256 8192 > gpurun_out/r2d_tl_cfg3.txt 2>&1
timeout -s KILL 600 python -m pytest tests/test_fused_step.py tests/test_gpu_parity.py -x -q > gpurun_out/r2d_tests.log 2>&1
tail -3 gpurun_out/r2d_tests.log
timeout -s KILL 300 python bench.py --config cfg2 --no-cpu-baseline --no-e2e > gpurun_out/r2d_bench_cfg2.json 2> gpurun_out/r2d_bench_cfg2.err
timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2d_bench_cfg3.json 2> gpurun_out/r2d_bench_cfg3.err
cat gpurun_out/r2d_tl_*.txt
