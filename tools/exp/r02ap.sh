#!/bin/bash
O=gpurun_out/r02ap; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_parity.py tests/test_gpu_cdr.py tests/test_gpu_generic.py -q -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
tail -n 3 $O/tests.log
for i in 1 2; do
  timeout 600 python bench.py --no-cpu > $O/bench_$i.json 2>> $O/bench.err
  python -c "import json;d=json.load(open('$O/bench_$i.json'));print('c1 value',d['value'],'e2e',d['e2e']['value'])"
done
timeout 600 python bench.py --no-cpu --config c4 > $O/bench_c4.json 2>> $O/bench.err
python -c "import json;d=json.load(open('$O/bench_c4.json'));print('c4 value',d['value'],'e2e',d['e2e']['value'])"
