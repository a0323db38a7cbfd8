set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/g1_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/g1_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/g1_bench.json
python tools/kbench.py --members 64 --sweeps 63 --reps 2 > gpurun_out/g1_kb.log 2>&1; tail -2 gpurun_out/g1_kb.log
