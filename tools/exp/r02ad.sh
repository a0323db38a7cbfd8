#!/bin/bash
# strided-DMA f upload / u download (BP_DMA2D) A/B on the c1 e2e line + the full GPU suite
O=gpurun_out/r02ad; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
tail -n 5 $O/gpu_tests.log
for v in 1 0 1 0; do
  BP_DMA2D=$v timeout 600 python bench.py --no-cpu > $O/bench_dma$v.json 2>> $O/bench.err
  python -c "import json;d=json.load(open('$O/bench_dma$v.json'));print('DMA2D=$v value',d['value'],'e2e',d['e2e']['value'],d['clocks']['sm_mhz'])"
done
