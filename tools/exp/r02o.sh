#!/bin/bash
O=gpurun_out/r02o; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_generic.py -q > $O/generic_tests.log 2>&1; echo "rc=$?" >> $O/generic_tests.log
timeout 900 python -m pytest tests/test_gpu_tri.py tests/test_gpu_cdr.py tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_slab.py -q -x > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 600 python bench.py --config c2 --slab --no-cpu > $O/bench_c2_slab.json 2> $O/bench_c2_slab.err
timeout 600 python bench.py --config c2 --slab --fused --no-cpu > $O/bench_c2_slab_fused.json 2> $O/bench_c2_slab_fused.err
