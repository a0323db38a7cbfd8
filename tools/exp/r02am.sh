#!/bin/bash
O=gpurun_out/r02am; mkdir -p $O
for v in base clw8 base clw8; do
  if [ $v = base ]; then unset BP_LIB_PATH; else export BP_LIB_PATH=variants/$v/libbornsweep.so; fi
  echo "== $v" >> $O/kbench.log
  timeout 300 python tools/kbench.py --config c2 --members 1 --sweeps 64 --reps 2 >> $O/kbench.log 2>&1
done
export BP_LIB_PATH=variants/clw8/libbornsweep.so
timeout 600 python -m pytest tests/test_gpu_tri.py tests/test_gpu_long.py -q -x > $O/tests_clw8.log 2>&1; echo "rc=$?" >> $O/tests_clw8.log
tail -n 3 $O/tests_clw8.log
cat $O/kbench.log
