# One GPU call that refreshes the round's evidence: bench lines, ncu launch lists and --set full captures.
# usage: bash tools/profile_round.sh TAG   (outputs under gpurun_out/TAG_*; summarise with tools/ncu_summary.py)
set -u
T=${1:-rx}
mkdir -p gpurun_out
K="regex:select|persist|greedy|compact|finalize|rowmap"
timeout -s KILL 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
for c in cfg3g cfg1 cfg2; do
  timeout -s KILL 300 python bench.py --config $c > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
done
timeout -s KILL 600 python bench.py --config cfg4 > gpurun_out/${T}_bench_cfg4.json 2> gpurun_out/${T}_bench_cfg4.err
for c in cfg3 cfg3g; do
  timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 24 --csv \
    --log-file gpurun_out/${T}_launches_$c.csv python bench.py --config $c --steps 8 --warmup 4 --no-graph \
    --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:persist_stream -c 1 \
  -o gpurun_out/${T}_stream python bench.py --config cfg3 --steps 3 --warmup 3 --no-graph --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:select1 -c 1 \
  -o gpurun_out/${T}_select python bench.py --config cfg3 --steps 3 --warmup 3 --no-graph --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:persist_greedy -c 1 \
  -o gpurun_out/${T}_greedy python bench.py --config cfg3g --steps 3 --warmup 3 --no-graph --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out | grep ${T}_
# latency-bound configs: every kernel of one step, full sets (cfg2 = BASELINE configs[1], cfg1 = configs[0])
for c in cfg2 cfg1; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "$K" -c 4 \
    -o gpurun_out/${T}_full_$c python bench.py --config $c --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-e2e > /dev/null 2>&1
  timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 24 --csv \
    --log-file gpurun_out/${T}_launches_$c.csv python bench.py --config $c --steps 8 --warmup 4 --no-graph \
    --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
timeout -s KILL 300 python bench.py --input logits > gpurun_out/${T}_bench_logits.json 2> gpurun_out/${T}_bench_logits.err
ls -la gpurun_out | grep ${T}_
