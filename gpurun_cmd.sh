mkdir -p gpurun_out/final3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final3/smoke.log 2>&1
timeout 1800 python -m pytest tests/ -m gpu -q 2>&1 | tail -4 > gpurun_out/final3/gpu_tests.log
timeout 900 python bench.py > gpurun_out/final3/bench_c1.json 2> gpurun_out/final3/bench_c1.err
tail -1 gpurun_out/final3/smoke.log; cat gpurun_out/final3/gpu_tests.log; tail -c 300 gpurun_out/final3/bench_c1.json
