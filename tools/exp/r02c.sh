#!/bin/bash
# A/B: row kernel before/after 9082168 (variants/old = e533695); ncu of the tridiagonal column pass
mkdir -p gpurun_out/r02c
for v in old main old main; do
  if [ $v = main ]; then export BP_LIB_PATH=; else export BP_LIB_PATH=variants/$v/libbornsweep.so; fi
  echo "== $v" >> gpurun_out/r02c/ab.log
  BP_COL_DST=1 timeout 300 python tools/kbench.py --members 64 --sweeps 63 --reps 2 >> gpurun_out/r02c/ab.log 2>&1
done
unset BP_LIB_PATH
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'tri_kernel' -s 2 -c 1 -o gpurun_out/r02c/tri python tools/profile_sweep.py --members 64 --sweeps 4 > gpurun_out/r02c/ncu.log 2>&1
