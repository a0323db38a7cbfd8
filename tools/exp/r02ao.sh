#!/bin/bash
O=gpurun_out/r02ao; mkdir -p $O
for d in 1 2 3; do
  timeout 600 python bench.py --no-cpu --e2e-depth $d > $O/bench_depth$d.json 2>> $O/bench.err
  python -c "import json;d=json.load(open('$O/bench_depth$d.json'));print('depth $d value',d['value'],'e2e',d['e2e']['value'])"
done
