#!/bin/bash
O=gpurun_out/r02bg; mkdir -p $O
timeout 900 python tools/exp/waves_stress.py 8 > $O/stress.log 2>&1
cat $O/stress.log | tail -12
