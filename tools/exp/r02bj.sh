#!/bin/bash
O=gpurun_out/r02bj; mkdir -p $O
timeout 900 python tools/exp/stagger_stress.py 8 > $O/stagger.log 2>&1
tail -n 30 $O/stagger.log
