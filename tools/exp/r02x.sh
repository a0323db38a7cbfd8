#!/bin/bash
O=gpurun_out/r02x; mkdir -p $O
for r in 1 2; do
timeout 600 python bench.py --no-cpu --steps 10 > $O/bench_c1_$r.json 2> $O/bench_c1_$r.err
BP_SPLIT=2 timeout 600 python bench.py --no-cpu --steps 10 > $O/bench_c1_split_$r.json 2> $O/bench_c1_split_$r.err
done
