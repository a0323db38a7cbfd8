python tools/profile_sweep.py --members 64 --sweeps 4 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'row_kernel<\(int\)9, \(int\)3|col_kernel' -s 2 -c 2 -o gpurun_out/prof3 python tools/profile_sweep.py --members 64 --sweeps 4 > gpurun_out/ncu.log 2>&1
python tools/profile_sweep.py --config c4 --members 32 --sweeps 6 > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'crow_kernel<\(int\)10, \(int\)3|ccol_kernel<\(int\)10, \(int\)1' -s 2 -c 2 -o gpurun_out/prof3c4 python tools/profile_sweep.py --config c4 --members 32 --sweeps 6 > gpurun_out/ncu4.log 2>&1
