#!/bin/bash
# r02: validation + bench lines + profiles after the tridiagonal column pass
O=gpurun_out/r02k; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
for c in c2 c3 c4 c0; do timeout 600 python bench.py --config $c --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --no-cpu --steps 2 --warmup 3 > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'tri_kernel|row_kernel' -s 4 -c 2 -o $O/c1_full python tools/profile_sweep.py --members 64 --sweeps 4 > $O/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'tri_kernel' -s 2 -c 1 -o $O/c2_tri python tools/profile_sweep.py --config c2 --members 1 --sweeps 4 > $O/ncu_c2.log 2>&1
