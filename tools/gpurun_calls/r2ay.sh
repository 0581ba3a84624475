# final code: synccheck / racecheck over tools/sanitize.py, ncu --set full of the one-launch kernels (cfg2, cfg1)
mkdir -p gpurun_out
for t in synccheck racecheck; do
  timeout -s KILL 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py > gpurun_out/r2j_$t.txt 2>&1
  echo "== $t"; tail -2 gpurun_out/r2j_$t.txt
done
K="regex:select|persist|greedy|compact|finalize|rowmap"
for c in cfg2 cfg1; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "$K" -c 4 \
    -o gpurun_out/r2j_full_$c python bench.py --config $c --steps 2 --warmup 3 --no-graph --no-cpu-baseline --no-e2e > /dev/null 2>&1
  timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 24 --csv \
    --log-file gpurun_out/r2j_launches_$c.csv python bench.py --config $c --steps 8 --warmup 4 --no-graph \
    --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
ls -la gpurun_out | grep r2j_
