#!/bin/bash
# group-major waves (BP_GROUP members per wave, BP_SPLIT parts per wave): c1 A/B
O=gpurun_out/r02as; mkdir -p $O
for cfg in "0 2" "8 4" "8 2" "16 4" "16 2" "32 4" "32 2" "4 2" "0 2"; do
  set -- $cfg
  BP_GROUP=$1 BP_SPLIT=$2 timeout 300 python bench.py --no-cpu --steps 10 > $O/bench_g$1_s$2.json 2>> $O/bench.err
  python -c "import json;d=json.load(open('$O/bench_g$1_s$2.json'));print('GROUP=$1 SPLIT=$2 value',round(d['value'],3),'e2e',round(d['e2e']['value'],3),d['clocks']['sm_mhz'])"
done
