#!/bin/bash
# after pruning the slower variants + tridiagonal slab column pass: GPU suite, slab kbench
O=gpurun_out/r02l; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 600 python bench.py --config c2 --slab --no-cpu > $O/bench_c2_slab.json 2> $O/bench_c2_slab.err
timeout 600 python bench.py --config c2 --slab --fused --no-cpu > $O/bench_c2_slab_fused.json 2> $O/bench_c2_slab_fused.err
timeout 600 python bench.py --config c3 --slab --no-cpu > $O/bench_c3_slab.json 2> $O/bench_c3_slab.err
