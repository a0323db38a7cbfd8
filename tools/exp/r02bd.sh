#!/bin/bash
O=gpurun_out/r02bd; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_determinism.py -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
grep -E "^FAILED|passed|failed|^E  |rc=" $O/tests.log | head
