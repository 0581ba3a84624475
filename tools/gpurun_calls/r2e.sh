mkdir -p gpurun_out
timeout -s KILL 300 python tools/dbg_stream.py 256 8 32000 1024 > gpurun_out/r2e_tl_cfg2_fused.txt 2>&1
TETRIS_NO_FUSED=1 timeout -s KILL 300 python tools/dbg_stream.py 256 8 32000 1024 > gpurun_out/r2e_tl_cfg2_plain.txt 2>&1
cat gpurun_out/r2e_tl_*.txt
