#!/bin/bash
# r02 validation of HEAD: GPU tests, smoke, c1 bench, reference arm
mkdir -p gpurun_out/r02a
nvidia-smi > gpurun_out/r02a/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02a/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02a/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r02a/bench.json 2> gpurun_out/r02a/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02a/bench_ref.json 2> gpurun_out/r02a/bench_ref.err
