for v in main nopersist; do
  if [ $v = main ]; then export BP_LIB_PATH=; else export BP_LIB_PATH=variants/$v/libbornsweep.so; fi
  echo "== $v"; timeout 300 python tools/kbench.py --members 64 --sweeps 63 --reps 2 2>&1 | tail -1
  timeout 300 python tools/kbench.py --config c4 --members 32 --sweeps 31 --reps 2 2>&1 | tail -1
done
unset BP_LIB_PATH
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
