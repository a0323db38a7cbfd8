#!/bin/bash
# wide-tile cluster tridiagonal pass (n >= 2048): parity, then c2 A/B
O=gpurun_out/r02ak; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tri.py tests/test_gpu_long.py tests/test_gpu_determinism.py -q -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
grep -E "^FAILED|passed|failed|^E  |rc=" $O/tests.log | head -20
for v in 1 0 1 0; do
  echo "== BP_TRI_WIDE=$v" >> $O/kbench.log
  BP_TRI_WIDE=$v timeout 300 python tools/kbench.py --config c2 --members 1 --sweeps 64 --reps 2 >> $O/kbench.log 2>&1
done
cat $O/kbench.log
