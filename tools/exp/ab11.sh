for rep in 1 2; do for v in main gsel orig; do
  if [ $v = main ]; then export BP_LIB_PATH=; else export BP_LIB_PATH=variants/$v/libbornsweep.so; fi
  echo "== $v"; timeout 300 python tools/kbench.py --members 64 --sweeps 63 --reps 2 2>&1 | tail -1
done; done
