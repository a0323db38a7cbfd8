for mx in 0 1; do
  echo "== MIXED=$mx"; BP_MIXED=$mx timeout 300 python tools/kbench.py --members 64 --sweeps 63 --reps 2 2>&1 | tail -1
done
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
