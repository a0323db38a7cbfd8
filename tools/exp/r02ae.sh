#!/bin/bash
# tiled T layout for n >= 2048: parity at 2048 / 4096, c2 bench; OptimalScalar n = 256 drift diagnostic;
# e2e amortisation with 45 steps
O=gpurun_out/r02ae; mkdir -p $O
timeout 600 python tools/exp/diag_opt256.py > $O/diag_opt256.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tri.py tests/test_gpu_long.py tests/test_gpu_slab.py -q -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -n 6 $O/tests.log
timeout 600 python bench.py --config c2 --no-cpu > $O/bench_c2.json 2> $O/bench_c2.err
python -c "import json;d=json.load(open('$O/bench_c2.json'));print('c2 value',d['value'],'e2e',d['e2e']['value'],d['roofline'])"
timeout 600 python bench.py --no-cpu --steps 45 > $O/bench_c1_45.json 2> $O/bench_c1_45.err
python -c "import json;d=json.load(open('$O/bench_c1_45.json'));print('c1 45 steps value',d['value'],'e2e',d['e2e']['value'])"
cat $O/diag_opt256.log
