#!/bin/bash
O=gpurun_out/r02bl; mkdir -p $O
for i in 1 2; do
timeout 300 python bench.py --no-cpu --steps 15 > $O/bench_$i.json 2>> $O/bench.err
python -c "import json;d=json.load(open('$O/bench_$i.json'));r=d['roofline'];print('value',round(d['value'],3),'e2e',round(d['e2e']['value'],3),'row',round(r['avg_launch_ms'],4),round(r['frac'],3),'col',round(r['column_kernel']['avg_launch_ms'],4),round(r['column_kernel']['frac'],3),'sweep',round(r['sweep']['frac'],3),'timed',round(r['sweep']['timed_region']['frac'],3),'instr',round(d['value_instrumented'],2))"
done
timeout 300 python tools/kbench.py --config c1 --members 64 --sweeps 127 --reps 2 2>&1 | tail -n 2
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -q 2>&1 | tail -n 2
