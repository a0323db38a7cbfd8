#!/bin/bash
O=gpurun_out/r02az; mkdir -p $O
for v in base l2h0 l2h5 base; do
  if [ $v = base ]; then unset BP_LIB_PATH; else export BP_LIB_PATH=variants/$v/libbornsweep.so; fi
  timeout 300 python bench.py --no-cpu --steps 10 > $O/bench_$v.json 2>> $O/bench.err
  python -c "import json;d=json.load(open('$O/bench_$v.json'));print('$v value',round(d['value'],3),'e2e',round(d['e2e']['value'],3),d['clocks']['sm_mhz'])"
done
unset BP_LIB_PATH
for cfg in "10 10" "12 12" "16 16" "9 9" "8 8"; do
  set -- $cfg
  BP_GROUP=$1 BP_SPLIT=$2 timeout 300 python bench.py --no-cpu --steps 10 > $O/bench_g$1.json 2>> $O/bench.err
  python -c "import json;d=json.load(open('$O/bench_g$1.json'));print('hints=1 GROUP=$1 SPLIT=$2 value',round(d['value'],3),'e2e',round(d['e2e']['value'],3))"
done
for c in c2 c3; do timeout 600 python bench.py --config $c --no-cpu --steps 8 > $O/bench_$c.json 2>> $O/bench.err
python -c "import json;d=json.load(open('$O/bench_$c.json'));print('$c value',round(d['value'],3),'e2e',round(d['e2e']['value'],3))"; done
