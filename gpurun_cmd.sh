mkdir -p gpurun_out/r2q
timeout 900 python -m pytest tests/test_gpu_bench_kernels.py -x -q -k "not full_size and not downscaled" > gpurun_out/r2q/tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2q/tests.log
MCQ_Z2PERSIST=x timeout 900 python -m pytest tests/test_gpu_slabs.py -x -q > gpurun_out/r2q/tests2.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2q/tests2.log
for v in base np_ldg p_tma; do
  L=""; [ $v != base ] && L=variants/$v.so
  MCQ_LIB_PATH=$L python bench.py --config 1 --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r2q/${v}_c1.json 2> gpurun_out/r2q/${v}_c1.err
  MCQ_LIB_PATH=$L python bench.py --config 4 --steps 12 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r2q/${v}_c4.json 2> gpurun_out/r2q/${v}_c4.err
done
tail -2 gpurun_out/r2q/tests.log gpurun_out/r2q/tests2.log
