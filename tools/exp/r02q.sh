#!/bin/bash
O=gpurun_out/r02q; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_cluster.py -q -x > $O/cluster_tests.log 2>&1; echo "rc=$?" >> $O/cluster_tests.log
timeout 300 python bench.py --config c0 --no-cpu > $O/bench_c0.json 2> $O/bench_c0.err
BP_CLUSTER=0 timeout 300 python bench.py --config c0 --no-cpu > $O/bench_c0_noclu.json 2> $O/bench_c0_noclu.err
