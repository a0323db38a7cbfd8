python -m pytest tests/test_gpu_periodic.py tests/test_gpu_direct.py tests/test_gpu_pipeline.py -q -x > gpurun_out/g2_tests.log 2>&1; echo "new tests rc=$?"
tail -15 gpurun_out/g2_tests.log
python -m pytest tests -m gpu -q > gpurun_out/g2_all.log 2>&1; echo "all rc=$?"; tail -3 gpurun_out/g2_all.log
