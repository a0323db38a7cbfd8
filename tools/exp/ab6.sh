export BP_MIXED=0
for v in main r85 r85pd3; do
  if [ $v = main ]; then export BP_LIB_PATH=; else export BP_LIB_PATH=variants/$v/libbornsweep.so; fi
  echo "== $v"; timeout 300 python tools/kbench.py --members 64 --sweeps 63 --reps 2 2>&1 | tail -1
done
unset BP_LIB_PATH
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
