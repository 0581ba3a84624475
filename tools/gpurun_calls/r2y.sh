mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_dist_gpu.py -x -q > gpurun_out/r2y_tests.log 2>&1
tail -30 gpurun_out/r2y_tests.log
