#!/bin/bash
O=gpurun_out/r02aj; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_cdr.py -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
grep -E "^FAILED|passed|failed|^E  " $O/tests.log | head -40
