#!/bin/bash
O=gpurun_out/r02n; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 600 python bench.py --config c2 --slab --no-cpu > $O/bench_c2_slab.json 2> $O/bench_c2_slab.err
timeout 600 python bench.py --config c2 --slab --fused --no-cpu > $O/bench_c2_slab_fused.json 2> $O/bench_c2_slab_fused.err
