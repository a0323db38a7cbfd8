#!/bin/bash
# CDR tridiagonal pass + full GPU suite (incl. long fixtures present) + sanitizers + c4 bench
O=gpurun_out/r02m; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_tri.py -x -q > $O/tri_tests.log 2>&1; echo "rc=$?" >> $O/tri_tests.log
timeout 300 python tools/kbench.py --config c4 --members 32 --sweeps 31 --reps 2 > $O/kb_c4.log 2>&1
BP_COL_DST=1 timeout 300 python tools/kbench.py --config c4 --members 32 --sweeps 31 --reps 1 >> $O/kb_c4.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 600 python bench.py --config c4 --no-cpu > $O/bench_c4.json 2> $O/bench_c4.err
