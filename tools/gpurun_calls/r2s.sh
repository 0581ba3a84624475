# latency-bound configs with the one-launch steps: per-CTA timelines + ncu full captures
mkdir -p gpurun_out
K="regex:select|persist|greedy|compact|finalize|rowmap"
timeout -s KILL 300 python tools/dbg_stream.py 256 8 32000 1024 > gpurun_out/r2s_tl_cfg2.txt 2>&1
timeout -s KILL 300 python tools/dbg_greedy.py 16 5 32000 48 > gpurun_out/r2s_tl_cfg1.txt 2>&1
for c in cfg2 cfg1; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "$K" -c 2 \
    -o gpurun_out/r2s_full_$c python bench.py --config $c --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-e2e > /dev/null 2>&1
  timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 24 --csv \
    --log-file gpurun_out/r2s_launches_$c.csv python bench.py --config $c --steps 8 --warmup 4 --no-graph \
    --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
cat gpurun_out/r2s_tl_*.txt
ls -la gpurun_out | grep r2s_
