mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2a_smoke.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_gpu_tests.log 2>&1
tail -3 gpurun_out/r2a_gpu_tests.log
timeout -s KILL 400 python bench.py --impl reference > gpurun_out/r2a_bench_ref.json 2> gpurun_out/r2a_bench_ref.err
bash tools/profile_round.sh r2a
