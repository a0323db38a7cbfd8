python tools/profile_sweep.py --members 64 --sweeps 4 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'row_kernel<\(int\)9, \(int\)3' -s 1 -c 1 -o gpurun_out/prof_row python tools/profile_sweep.py --members 64 --sweeps 4 > gpurun_out/ncu.log 2>&1
