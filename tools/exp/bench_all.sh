python bench.py > gpurun_out/b_c1.log 2>&1
for c in c4 c2 c3 c0; do python bench.py --config $c --no-cpu > gpurun_out/b_$c.log 2>&1; done
