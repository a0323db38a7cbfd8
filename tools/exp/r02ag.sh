#!/bin/bash
# c1 row kernel + tri kernel: source-level ncu of the current build
O=gpurun_out/r02ag; mkdir -p $O
K="--set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 ncu $K -k regex:'row_kernel<\(int\)9, \(int\)3|tri_kernel<\(int\)9' -s 2 -c 2 -o $O/c1 python tools/profile_sweep.py --config c1 --members 64 --sweeps 4 > $O/ncu_c1.log 2>&1
tail -n 3 $O/ncu_c1.log
