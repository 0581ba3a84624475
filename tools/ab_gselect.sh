for v in libA.so libtetris_b200.so; do
  for w in 4 8; do TETRIS_LIB_VARIANT=$v timeout -s KILL 300 python bench.py --simulate-world $w --steps 500 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$v W=$w\", round(d[\"ms_per_step\"]*1000,2))"; done
  TETRIS_LIB_VARIANT=$v timeout -s KILL 300 python bench.py --config cfg4 --steps 300 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$v cfg4\", {k: round(v['us_per_select'],2) for k,v in d['sweep'].items()})"
done
