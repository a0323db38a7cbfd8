for mx in 1 0; do
  echo "== BP_MIXED=$mx"; BP_MIXED=$mx timeout 300 python tools/kbench.py --members 64 --sweeps 63 --reps 3 2>&1 | tail -1
  BP_MIXED=$mx timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 | cut -c1-300
done
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
