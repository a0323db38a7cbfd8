for pp in 16 8; do for mx in 0 1; do
  echo "== PP=$pp MIXED=$mx"; BP_POINTS_PER_THREAD=$pp BP_MIXED=$mx timeout 300 python tools/kbench.py --members 64 --sweeps 63 --reps 2 2>&1 | tail -1
done; done
