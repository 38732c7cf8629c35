mkdir -p gpurun_out/v6
timeout 600 python -m pytest tests/test_gpu_thermal.py -q -m gpu > gpurun_out/v6/tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/v6/tests.log
tail -n 15 gpurun_out/v6/tests.log
