#!/bin/bash
O=gpurun_out/r02av; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_parity.py tests/test_gpu_long.py tests/test_gpu_pipeline.py -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -n 3 $O/tests.log
for b in 64 32 16 8; do
  for cfg in "default" "0 x"; do
    set -- $cfg
    if [ $1 = default ]; then unset BP_GROUP; else export BP_GROUP=$1; fi
    timeout 300 python bench.py --no-cpu --steps 10 --batch $b > $O/bench_b${b}_$1.json 2>> $O/bench.err
    python -c "import json;d=json.load(open('$O/bench_b${b}_$1.json'));print('batch $b GROUP=$1 value',round(d['value'],3),'e2e',round(d['e2e']['value'],3),d['clocks']['sm_mhz'])"
  done
done
unset BP_GROUP
BP_SPLIT=8 timeout 300 python bench.py --no-cpu --steps 10 --batch 8 > $O/bench_b8_s8.json 2>> $O/bench.err
python -c "import json;d=json.load(open('$O/bench_b8_s8.json'));print('batch 8 SPLIT=8 value',round(d['value'],3),'e2e',round(d['e2e']['value'],3))"
BP_SPLIT=8 timeout 300 python bench.py --no-cpu --steps 10 --batch 16 > $O/bench_b16_s8.json 2>> $O/bench.err
python -c "import json;d=json.load(open('$O/bench_b16_s8.json'));print('batch 16 (waves of 8) SPLIT=8 value',round(d['value'],3),'e2e',round(d['e2e']['value'],3))"
