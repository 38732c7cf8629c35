mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_trace.py -q -x -k sweep --durations=3 2>&1 | tail -30 > gpurun_out/t65.log
cat gpurun_out/t65.log
