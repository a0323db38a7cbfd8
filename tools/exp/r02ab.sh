#!/bin/bash
# staged maps on slabs: slab GPU tests first, then the full suite, then the c1 bench line
O=gpurun_out/r02ab; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_slab.py -q -x > $O/slab_tests.log 2>&1; echo "rc=$?" >> $O/slab_tests.log
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
tail -3 $O/slab_tests.log $O/gpu_tests.log; cat $O/bench.json | head -c 600
