set -x
mkdir -p gpurun_out/th
timeout 600 python -m pytest tests/test_gpu_thermal.py tests/test_gpu_parity.py -q -m gpu -k "thermal or Thermal or langevin or temperature or divergence" > gpurun_out/th/th.log 2>&1
timeout 900 python -m pytest tests/ -m gpu -q > gpurun_out/th/gpu_tests.log 2>&1
python bench.py --steps 200 --warmup 5 > gpurun_out/th/bench_c1.json 2> gpurun_out/th/bench_c1.err
tail -3 gpurun_out/th/th.log gpurun_out/th/gpu_tests.log
