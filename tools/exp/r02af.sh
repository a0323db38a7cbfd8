#!/bin/bash
# c2 tridiagonal pass: source-level ncu (where does the tile loop stall?); OptimalScalar drift diagnostic
O=gpurun_out/r02af; mkdir -p $O
timeout 600 python tools/exp/diag_opt256.py > $O/diag_opt256.log 2>&1
K="--set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 ncu $K -k regex:'tri_kernel<\(int\)12' -s 2 -c 1 -o $O/c2tri python tools/profile_sweep.py --config c2 --members 1 --sweeps 4 > $O/ncu_c2.log 2>&1
cat $O/diag_opt256.log; tail -n 3 $O/ncu_c2.log
