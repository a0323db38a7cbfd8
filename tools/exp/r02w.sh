#!/bin/bash
O=gpurun_out/r02w; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_cluster.py tests/test_gpu_parity.py -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for b in 8 16 32; do
  timeout 600 python bench.py --batch $b --no-cpu --steps 8 > $O/bench_b$b.json 2> $O/bench_b$b.err
  BP_SPLIT=0 timeout 600 python bench.py --batch $b --no-cpu --steps 8 > $O/bench_b${b}_nosplit.json 2> $O/bench_b${b}_nosplit.err
done
