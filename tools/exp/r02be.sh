#!/bin/bash
O=gpurun_out/r02be; mkdir -p $O
for cfg in "0 2" "4 4" "8 8" "8 4" "6 6" "16 8" "2 2" "0 2"; do
  set -- $cfg
  BP_GROUP=$1 BP_SPLIT=$2 timeout 300 python bench.py --config c4 --no-cpu --steps 10 --e2e-depth 1 > $O/bench_c4_g$1_s$2.json 2>> $O/bench.err
  python -c "import json;d=json.load(open('$O/bench_c4_g$1_s$2.json'));print('c4 GROUP=$1 SPLIT=$2 value',round(d['value'],3),d['clocks']['sm_mhz'])"
done
timeout 300 python -m pytest tests/test_gpu_cdr.py tests/test_gpu_determinism.py -q 2>&1 | tail -n 2
