#!/bin/bash
# row kernel: L2 prefetch of the T lines BS_ROW_PF_AHEAD groups ahead (A/B on c1)
O=gpurun_out/r02ah; mkdir -p $O
for v in base pf148 pf296 base pf148 pf296; do
  if [ $v = base ]; then unset BP_LIB_PATH; else export BP_LIB_PATH=variants/$v/libbornsweep.so; fi
  echo "== $v" >> $O/kbench.log
  timeout 300 python tools/kbench.py --config c1 --members 64 --sweeps 127 --reps 3 >> $O/kbench.log 2>&1
done
cat $O/kbench.log
