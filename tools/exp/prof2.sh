export BP_MIXED=0
python tools/profile_sweep.py --members 64 --sweeps 4 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'row_kernel<\(int\)9, \(int\)3|col_kernel' -s 2 -c 2 -o gpurun_out/prof2 python tools/profile_sweep.py --members 64 --sweeps 4 > gpurun_out/ncu.log 2>&1
