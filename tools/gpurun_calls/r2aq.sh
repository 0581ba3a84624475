# final-code evidence (r2h): the full GPU suite, smoke, the round's bench lines and ncu captures (tools/profile_round.sh)
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests/ -q -m gpu > gpurun_out/r2h_gpu_tests.log 2>&1
tail -2 gpurun_out/r2h_gpu_tests.log
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/profile_round.sh r2h
