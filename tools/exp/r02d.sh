#!/bin/bash
# A/B: row kernel old / main (inv_eta hoisted) / noinv; tri column pass after the bank-conflict fix
mkdir -p gpurun_out/r02d
for v in old main noinv old main noinv; do
  if [ $v = main ]; then export BP_LIB_PATH=; else export BP_LIB_PATH=variants/$v/libbornsweep.so; fi
  echo "== $v" >> gpurun_out/r02d/ab.log
  timeout 300 python tools/kbench.py --members 64 --sweeps 63 --reps 2 >> gpurun_out/r02d/ab.log 2>&1
done
unset BP_LIB_PATH
timeout 300 python tools/kbench.py --config c2 --members 1 --sweeps 63 --reps 2 >> gpurun_out/r02d/ab.log 2>&1
timeout 600 python -m pytest tests/test_gpu_tri.py -x -q > gpurun_out/r02d/tri_tests.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'tri_kernel' -s 2 -c 1 -o gpurun_out/r02d/tri python tools/profile_sweep.py --members 64 --sweeps 4 > gpurun_out/r02d/ncu.log 2>&1
