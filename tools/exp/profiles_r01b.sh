python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --no-cpu --steps 3 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
python tools/profile_sweep.py --members 64 --sweeps 4 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'row_kernel|col_kernel' -s 5 -c 2 -o gpurun_out/full_c1 python tools/profile_sweep.py --members 64 --sweeps 4 > gpurun_out/ncu_full.log 2>&1
