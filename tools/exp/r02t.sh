#!/bin/bash
O=gpurun_out/r02t; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py --batch 8 --no-cpu > $O/bench_c1_b8.json 2> $O/bench_c1_b8.err
timeout 900 ncu --set full --clock-control none -k regex:'row_kernel<.*, 3,|tri_kernel' -s 2 -c 2 -o $O/c2_full python tools/profile_sweep.py --config c2 --members 1 --sweeps 4 > $O/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:'row_kernel<.*, 3,|tri_kernel' -s 4 -c 2 -o $O/c3_full python tools/profile_sweep.py --config c3 --members 1 --sweeps 4 > $O/ncu_c3.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:'crow_kernel<.*, 2,|crow_kernel<.*, 3,|tri_kernel' -s 3 -c 3 -o $O/c4_full python tools/profile_sweep.py --config c4 --members 32 --sweeps 4 > $O/ncu_c4.log 2>&1
