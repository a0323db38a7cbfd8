#!/bin/bash
O=gpurun_out/r02bh; mkdir -p $O
BP_LIB_PATH=variants/old/libbornsweep.so timeout 900 python tools/exp/waves_stress.py 10 > $O/stress_old.log 2>&1
tail -n 11 $O/stress_old.log
