#!/bin/bash
O=gpurun_out/r02y; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_determinism.py -q -k split > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
BP_SPLIT=4 timeout 600 python -m pytest tests/test_gpu_determinism.py -q -k split >> $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for k in 2 3 4 2 3 4; do
BP_SPLIT=$k timeout 600 python bench.py --no-cpu --steps 10 > $O/bench_c1_k$k.json 2> $O/bench_c1_k$k.err
grep -h "^{" $O/bench_c1_k$k.json | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('k$k', round(d['value'],2), round(d['e2e']['value'],2), d['clocks']['sm_mhz'])" >> $O/summary.txt
done
for k in 2 4; do
BP_SPLIT=$k timeout 600 python bench.py --no-cpu --steps 8 --batch 8 > $O/bench_b8_k$k.json 2> $O/bench_b8_k$k.err
grep -h "^{" $O/bench_b8_k$k.json | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('b8 k$k', round(d['value'],2), round(d['e2e']['value'],2), d['clocks']['sm_mhz'])" >> $O/summary.txt
done
