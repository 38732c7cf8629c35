mkdir -p gpurun_out/r2h
timeout 1200 python -m pytest tests/test_gpu_bench_kernels.py -q -s > gpurun_out/r2h/tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2h/tests.log
python bench.py --config 1 --steps 400 --warmup 10 --no-cpu-baseline > gpurun_out/r2h/c1.json 2> gpurun_out/r2h/c1.err
python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2h/c4.json 2> gpurun_out/r2h/c4.err
python bench.py --config 1 --steps 8 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/r2h/plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_zconv2' -s 4 -c 1 -o gpurun_out/r2h/c1 python bench.py --config 1 --steps 8 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/r2h/ncu1.log 2>&1
python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/r2h/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_zconv2' -s 4 -c 1 -o gpurun_out/r2h/c4 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/r2h/ncu4.log 2>&1
grep -E "passed|failed|configs" gpurun_out/r2h/tests.log | tail -20
