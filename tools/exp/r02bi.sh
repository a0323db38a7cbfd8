#!/bin/bash
O=gpurun_out/r02bi; mkdir -p $O
timeout 900 python tools/exp/waves_stress.py 24 > $O/stress.log 2>&1
grep -c "mismatching members \[\] \[\]" $O/stress.log; grep -v "mismatching members \[\] \[\]" $O/stress.log | tail -n 8
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
tail -n 3 $O/gpu_tests.log
for i in 1 2; do
  timeout 300 python bench.py --no-cpu --steps 15 > $O/bench_$i.json 2>> $O/bench.err
  python -c "import json;d=json.load(open('$O/bench_$i.json'));print('value',round(d['value'],3),'e2e',round(d['e2e']['value'],3),d['clocks']['sm_mhz'])"
done
BP_GROUP=0 timeout 300 python bench.py --no-cpu --steps 10 > $O/bench_nowaves.json 2>> $O/bench.err
python -c "import json;d=json.load(open('$O/bench_nowaves.json'));print('no waves value',round(d['value'],3),'e2e',round(d['e2e']['value'],3))"
