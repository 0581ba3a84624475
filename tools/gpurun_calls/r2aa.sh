mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2aa_smoke.log 2>&1; tail -2 gpurun_out/r2aa_smoke.log
timeout -s KILL 2000 python -m pytest tests/ -x -q -m gpu > gpurun_out/r2aa_gpu_tests.log 2>&1
tail -3 gpurun_out/r2aa_gpu_tests.log
timeout -s KILL 400 python bench.py > gpurun_out/r2aa_bench.json 2> gpurun_out/r2aa_bench.err
tail -c 600 gpurun_out/r2aa_bench.json
