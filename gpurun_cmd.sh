mkdir -p gpurun_out/r2m
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_bench_kernels.py -x -q -k "not full_size" > gpurun_out/r2m/tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2m/tests.log
for v in base uswz0; do
  L=""; [ $v = uswz0 ] && L=variants/uswz0.so
  MCQ_LIB_PATH=$L python bench.py --config 1 --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r2m/${v}_c1.json 2> gpurun_out/r2m/${v}_c1.err
  MCQ_LIB_PATH=$L python bench.py --config 4 --steps 12 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r2m/${v}_c4.json 2> gpurun_out/r2m/${v}_c4.err
done
python bench.py --loopback 8 --steps 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r2m/lb8.json 2> gpurun_out/r2m/lb8.err
MCQ_SLAB_SERIAL=1 python bench.py --loopback 8 --steps 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r2m/lb8serial.json 2> gpurun_out/r2m/lb8serial.err
python bench.py --config 1 --steps 8 --warmup 3 --no-cpu-baseline --profile-steps 1 --e2e-steps 2 > gpurun_out/r2m/plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_update' -s 8 -c 1 -o gpurun_out/r2m/ku1 python bench.py --config 1 --steps 8 --warmup 3 --no-cpu-baseline --profile-steps 1 --e2e-steps 2 > gpurun_out/r2m/ncu1.log 2>&1
python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --profile-steps 1 --e2e-steps 2 > gpurun_out/r2m/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_update' -s 8 -c 1 -o gpurun_out/r2m/ku4 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --profile-steps 1 --e2e-steps 2 > gpurun_out/r2m/ncu4.log 2>&1
tail -3 gpurun_out/r2m/tests.log
