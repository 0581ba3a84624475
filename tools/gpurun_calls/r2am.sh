# compute-sanitizer over the final code (tools/sanitize.py: + cfg1 / cfg2 one-launch shapes)
mkdir -p gpurun_out
for t in memcheck synccheck racecheck; do
  timeout -s KILL 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py > gpurun_out/r2am_$t.txt 2>&1
  echo "== $t"; tail -4 gpurun_out/r2am_$t.txt
done
