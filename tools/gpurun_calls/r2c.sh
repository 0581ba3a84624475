mkdir -p gpurun_out
timeout -s KILL 300 python tools/dbg_stream.py 256 8 32000 1024 > gpurun_out/r2c_tl_cfg2_fused.txt 2>&1
TETRIS_NO_FUSED=1 timeout -s KILL 300 python tools/dbg_stream.py 256 8 32000 1024 > gpurun_out/r2c_tl_cfg2_plain.txt 2>&1
timeout -s KILL 300 python tools/dbg_stream.py 16 5 32000 48 > gpurun_out/r2c_tl_cfg1s_fused.txt 2>&1
timeout -s KILL 600 python -m pytest tests/test_fused_step.py -x -q > gpurun_out/r2c_fused_tests.log 2>&1
tail -3 gpurun_out/r2c_fused_tests.log
cat gpurun_out/r2c_tl_*.txt
