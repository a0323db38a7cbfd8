#!/bin/bash
O=gpurun_out/r02aa; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_cdr.py tests/test_gpu_tri.py -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for r in 1 2; do
timeout 600 python bench.py --config c4 --no-cpu --steps 10 > $O/bench_c4_$r.json 2> $O/bench_c4_$r.err
BP_SPLIT=0 timeout 600 python bench.py --config c4 --no-cpu --steps 10 > $O/bench_c4_nosplit_$r.json 2> $O/bench_c4_nosplit_$r.err
done
