set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for m in 2 4 8 16 32 64; do timeout 300 python tools/kbench.py --members $m --sweeps 63 --reps 2 2>&1 | tail -1; done
for b in 4 8 16 64; do timeout 300 python bench.py --batch $b --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 | cut -c1-400; done
