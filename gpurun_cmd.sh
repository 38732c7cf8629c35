mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_trace.py -q -x --durations=5 -k bright 2>&1 | tail -30 > gpurun_out/gpu_tests53.log
cat gpurun_out/gpu_tests53.log
