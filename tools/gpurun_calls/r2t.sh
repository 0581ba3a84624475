mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_sim_gpu.py tests/test_gpu_parity.py -x -q -k "sim or cluster" > gpurun_out/r2t_tests.log 2>&1
tail -3 gpurun_out/r2t_tests.log
timeout -s KILL 600 python tools/bench_sim.py 1024 8 8 30 > gpurun_out/r2t_sim_b1024.json 2> gpurun_out/r2t_sim.err
timeout -s KILL 600 python tools/bench_sim.py 64 4 4 60 > gpurun_out/r2t_sim_b64.json 2>> gpurun_out/r2t_sim.err
cat gpurun_out/r2t_sim_*.json; tail -5 gpurun_out/r2t_sim.err
