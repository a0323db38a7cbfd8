#!/bin/bash
O=gpurun_out/r02u; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_generic.py tests/test_gpu_periodic.py -q > $O/generic_tests.log 2>&1; echo "rc=$?" >> $O/generic_tests.log
for v in main etasm main etasm; do
  if [ $v = main ]; then export BP_LIB_PATH=; else export BP_LIB_PATH=variants/$v/libbornsweep.so; fi
  echo "== $v" >> $O/ab.log
  timeout 300 python tools/kbench.py --members 64 --sweeps 63 --reps 2 >> $O/ab.log 2>&1
done
unset BP_LIB_PATH
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k regex:'row_kernel<12, 3' -s 2 -c 1 -o $O/c2_row python tools/profile_sweep.py --config c2 --members 1 --sweeps 4 > $O/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k regex:'row_kernel<8, 3' -s 2 -c 1 -o $O/c3_row python tools/profile_sweep.py --config c3 --members 1 --sweeps 4 > $O/ncu_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k regex:'crow_kernel<10, [23]' -s 2 -c 2 -o $O/c4_row python tools/profile_sweep.py --config c4 --members 32 --sweeps 4 > $O/ncu_c4.log 2>&1
