for b in 64 32 16; do
  st=$((40*64/b))
  python bench.py --no-cpu --batch $b --steps $st --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('batch $b', round(d['value'],3), d['clocks'], round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['column_kernel']['avg_launch_ms'],4))"
done
