#!/bin/bash
O=gpurun_out/r02bc; mkdir -p $O
for v in base gs32 base gs32; do
  if [ $v = base ]; then unset BP_LIB_PATH; else export BP_LIB_PATH=variants/$v/libbornsweep.so; fi
  timeout 300 python bench.py --no-cpu --steps 10 > $O/bench_$v.json 2>> $O/bench.err
  python -c "import json;d=json.load(open('$O/bench_$v.json'));print('$v value',round(d['value'],3),'e2e',round(d['e2e']['value'],3),d['clocks']['sm_mhz'])"
done
