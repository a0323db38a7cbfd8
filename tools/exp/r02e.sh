#!/bin/bash
mkdir -p gpurun_out/r02e
timeout 600 python -m pytest tests/test_gpu_tri.py -x -q > gpurun_out/r02e/tri_tests.log 2>&1
for cfg in c1 c2 c3 c0; do
  m=64; [ $cfg != c1 ] && m=1
  timeout 300 python tools/kbench.py --config $cfg --members $m --sweeps 63 --reps 2 >> gpurun_out/r02e/kb.log 2>&1
  BP_COL_DST=1 timeout 300 python tools/kbench.py --config $cfg --members $m --sweeps 63 --reps 1 >> gpurun_out/r02e/kb.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02e/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02e/gpu_tests.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'tri_kernel' -s 2 -c 1 -o gpurun_out/r02e/tri python tools/profile_sweep.py --members 64 --sweeps 4 > gpurun_out/r02e/ncu.log 2>&1
