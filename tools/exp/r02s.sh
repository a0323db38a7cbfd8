#!/bin/bash
O=gpurun_out/r02s; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_cluster.py -q -x > $O/cluster_tests.log 2>&1; echo "rc=$?" >> $O/cluster_tests.log
timeout 300 python bench.py --config c0 --no-cpu > $O/bench_c0.json 2> $O/bench_c0.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'cluster_solve' -c 1 -o $O/c0 python bench.py --config c0 --no-cpu --steps 1 --warmup 3 > $O/ncu.log 2>&1
