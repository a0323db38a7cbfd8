#!/bin/bash
O=gpurun_out/r02an; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_tri.py -q -x -k "wide" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -n 4 $O/tests.log
for v in 1 0 1 0; do
  BP_TRI_WIDE=$v timeout 600 python bench.py --config c2 --no-cpu > $O/bench_c2_wide$v.json 2>> $O/bench.err
  python -c "import json;d=json.load(open('$O/bench_c2_wide$v.json'));r=d['roofline'];print('WIDE=$v value',d['value'],'e2e',d['e2e']['value'],'col',r['column_kernel']['avg_launch_ms'],r['column_kernel']['frac'],'sweep',r['sweep']['frac'])"
done
