#!/bin/bash
O=gpurun_out/r02v; mkdir -p $O
K="--set full --clock-control none --kernel-name-base demangled"
timeout 900 ncu $K -k regex:'row_kernel<\(int\)12, \(int\)3|tri_kernel<\(int\)12' -s 2 -c 2 -o $O/c2 python tools/profile_sweep.py --config c2 --members 1 --sweeps 4 > $O/ncu_c2.log 2>&1
timeout 900 ncu $K -k regex:'row_kernel<\(int\)8, \(int\)3|tri_kernel<\(int\)8' -s 2 -c 2 -o $O/c3 python tools/profile_sweep.py --config c3 --members 1 --sweeps 4 > $O/ncu_c3.log 2>&1
timeout 900 ncu $K -k regex:'crow_kernel<\(int\)10, \(int\)[23]|tri_kernel<\(int\)10' -s 3 -c 3 -o $O/c4 python tools/profile_sweep.py --config c4 --members 32 --sweeps 4 > $O/ncu_c4.log 2>&1
