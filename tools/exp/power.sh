nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 100 > gpurun_out/power.csv &
SMI=$!
python bench.py --no-cpu --steps 40 --warmup 3 > gpurun_out/bench_long.log 2>&1
kill $SMI
