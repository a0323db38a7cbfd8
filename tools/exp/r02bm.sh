#!/bin/bash
O=gpurun_out/r02bm; mkdir -p $O
for i in 1 2; do
timeout 300 python bench.py --no-cpu --steps 15 > $O/bench_$i.json 2>> $O/bench.err
python -c "import json;d=json.load(open('$O/bench_$i.json'));r=d['roofline'];print('value',round(d['value'],3),'e2e',round(d['e2e']['value'],3),'row',round(r['avg_launch_ms'],4),round(r['frac'],3),'col',round(r['column_kernel']['avg_launch_ms'],4),round(r['column_kernel']['frac'],3),'sweep',round(r['sweep']['frac'],3),'timed',round(r['sweep']['timed_region']['frac'],3))"
done
timeout 300 python bench.py --no-cpu --steps 10 --batch 8 > $O/bench_b8.json 2>> $O/bench.err
python -c "import json;d=json.load(open('$O/bench_b8.json'));print('batch 8 value',round(d['value'],3),'e2e',round(d['e2e']['value'],3))"
for c in c2 c3; do timeout 600 python bench.py --config $c --no-cpu --steps 8 > $O/bench_$c.json 2>> $O/bench.err
python -c "import json;d=json.load(open('$O/bench_$c.json'));print('$c value',round(d['value'],3),'e2e',round(d['e2e']['value'],3))"; done
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
tail -n 3 $O/gpu_tests.log
