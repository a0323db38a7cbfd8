#!/bin/bash
# final state of the session: full GPU suite, smoke, bench lines, reference arm, launch list; c4 e2e depth
O=gpurun_out/r02l; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
for c in c2 c3 c4 c0; do timeout 600 python bench.py --config $c --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err; done
for d in 3 4; do timeout 600 python bench.py --config c4 --no-cpu --e2e-depth $d > $O/bench_c4_depth$d.json 2> $O/bench_c4_depth$d.err; done
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --no-cpu --steps 2 --warmup 3 > $O/ncu_launch.log 2>&1
tail -n 3 $O/gpu_tests.log; tail -n 1 $O/smoke.log
