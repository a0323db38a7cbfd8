timeout 300 python tools/kbench.py --members 64 --sweeps 63 --reps 2 2>&1 | tail -1
timeout 300 python tools/kbench.py --config c4 --members 32 --sweeps 31 --reps 2 2>&1 | tail -1
timeout 300 python tools/kbench.py --config c2 --members 1 --sweeps 31 --reps 2 2>&1 | tail -1
timeout 300 python tools/kbench.py --config c3 --members 1 --sweeps 31 --reps 2 2>&1 | tail -1
