mkdir -p gpurun_out/edge
timeout 1200 python -m pytest tests/test_gpu_edges.py -q -m gpu > gpurun_out/edge/edges.log 2>&1
tail -n 30 gpurun_out/edge/edges.log
