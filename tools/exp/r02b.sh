#!/bin/bash
# tridiagonal column pass: tests + kernel timing (tri vs transform route)
mkdir -p gpurun_out/r02b
timeout 600 python -m pytest tests/test_gpu_tri.py -x -q > gpurun_out/r02b/tri_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02b/tri_tests.log
for cfg in c1 c2; do
  m=64; [ $cfg = c2 ] && m=1
  timeout 300 python tools/kbench.py --config $cfg --members $m --sweeps 32 --reps 2 > gpurun_out/r02b/kb_${cfg}_tri.log 2>&1
  BP_COL_DST=1 timeout 300 python tools/kbench.py --config $cfg --members $m --sweeps 32 --reps 2 > gpurun_out/r02b/kb_${cfg}_dst.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02b/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02b/gpu_tests.log
