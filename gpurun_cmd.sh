mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dmi" 2>&1 | tail -5 > gpurun_out/t68.log
cat gpurun_out/t68.log
