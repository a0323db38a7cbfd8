#!/bin/bash
mkdir -p gpurun_out/r02j
for v in main stearly main stearly; do
  if [ $v = main ]; then export BP_LIB_PATH=; else export BP_LIB_PATH=variants/$v/libbornsweep.so; fi
  echo "== $v" >> gpurun_out/r02j/ab.log
  for cfg in c1 c2 c3; do
    m=64; [ $cfg != c1 ] && m=1
    timeout 300 python tools/kbench.py --config $cfg --members $m --sweeps 63 --reps 1 >> gpurun_out/r02j/ab.log 2>&1
  done
done
unset BP_LIB_PATH
timeout 600 python -m pytest tests/test_gpu_tri.py -x -q > gpurun_out/r02j/tri_tests.log 2>&1
