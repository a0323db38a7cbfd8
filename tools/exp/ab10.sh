for v in main r4 c4 r4c4; do
  if [ $v = main ]; then export BP_LIB_PATH=; else export BP_LIB_PATH=variants/$v/libbornsweep.so; fi
  echo "== $v"; timeout 300 python tools/kbench.py --members 64 --sweeps 63 --reps 2 2>&1 | tail -1
done
for v in main r4c4; do
  if [ $v = main ]; then export BP_LIB_PATH=; else export BP_LIB_PATH=variants/$v/libbornsweep.so; fi
  python bench.py --no-cpu --steps 30 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v bench', round(d['value'],3), d['clocks'], round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['column_kernel']['avg_launch_ms'],4))"
done
