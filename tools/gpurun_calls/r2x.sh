mkdir -p gpurun_out
for c in 4096 8192 32768 65536; do timeout -s KILL 120 python tools/dbg_gselect.py 4096 16 $c; done > gpurun_out/r2x_gsel.txt 2>&1
cat gpurun_out/r2x_gsel.txt
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:persist_stream -c 1 \
  -o gpurun_out/r2x_logits_stream python bench.py --input logits --steps 3 --warmup 3 --no-graph --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out | grep r2x
