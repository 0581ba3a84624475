# long fuzz run of the final kernels: 1000 randomised shapes through the product steps against the oracle
mkdir -p gpurun_out
TETRIS_FUZZ_DRAWS=1000 timeout -s KILL 2400 python -m pytest tests/test_fuzz_gpu.py -q -n 0 > gpurun_out/r2k_fuzz1000.log 2>&1 || \
TETRIS_FUZZ_DRAWS=1000 timeout -s KILL 2400 python -m pytest tests/test_fuzz_gpu.py -q > gpurun_out/r2k_fuzz1000.log 2>&1
tail -3 gpurun_out/r2k_fuzz1000.log
