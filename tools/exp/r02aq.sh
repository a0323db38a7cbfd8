#!/bin/bash
O=gpurun_out/r02aq; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_slab.py tests/test_gpu_direct.py tests/test_gpu_determinism.py -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
grep -E "^FAILED|passed|failed|^E  " $O/tests.log | head -30
