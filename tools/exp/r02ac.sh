#!/bin/bash
O=gpurun_out/r02ac; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_slab.py tests/test_gpu_determinism.py -q > $O/slab_tests.log 2>&1; echo "rc=$?" >> $O/slab_tests.log
tail -n 15 $O/slab_tests.log
