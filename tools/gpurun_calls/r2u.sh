mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_sim_gpu.py tests/test_dropin.py tests/test_gpu_parity.py -x -q -k "sim or stats or heap or dropin or select_tetris" > gpurun_out/r2u_tests.log 2>&1
tail -3 gpurun_out/r2u_tests.log
timeout -s KILL 600 python tools/bench_sim.py 1024 8 8 30 > gpurun_out/r2u_sim_b1024.json 2> gpurun_out/r2u_sim.err
cat gpurun_out/r2u_sim_*.json; tail -5 gpurun_out/r2u_sim.err
timeout -s KILL 300 python tools/dbg_greedy.py 16 5 32000 48 > gpurun_out/r2u_tl_cfg1.txt 2>&1; cat gpurun_out/r2u_tl_cfg1.txt
