#!/bin/bash
O=gpurun_out/r02ax; mkdir -p $O
timeout 900 python tools/exp/wave_scan.py > $O/wave_scan.log 2>&1
cat $O/wave_scan.log | tail -20
