#!/bin/bash
O=gpurun_out/r02al; mkdir -p $O
K="--set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 ncu $K -k regex:'tri_wide_kernel' -s 2 -c 1 -o $O/c2wide python tools/profile_sweep.py --config c2 --members 1 --sweeps 4 > $O/ncu_c2.log 2>&1
tail -n 3 $O/ncu_c2.log
