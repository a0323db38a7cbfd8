#!/bin/bash
O=gpurun_out/r02au; mkdir -p $O
for cfg in "8 8" "6 6" "10 10" "12 12" "16 16" "0 8" "0 16" "7 7" "9 9" "8 8"; do
  set -- $cfg
  BP_GROUP=$1 BP_SPLIT=$2 timeout 300 python bench.py --no-cpu --steps 10 > $O/bench_g$1_s$2.json 2>> $O/bench.err
  python -c "import json;d=json.load(open('$O/bench_g$1_s$2.json'));print('GROUP=$1 SPLIT=$2 value',round(d['value'],3),'e2e',round(d['e2e']['value'],3),d['clocks']['sm_mhz'])"
done
