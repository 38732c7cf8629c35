mkdir -p gpurun_out/r2j
for v in v3 v2 seq; do
  for c in 1 4; do
    st=200; [ $c = 4 ] && st=12
    MCQ_ZVARIANT=$v python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r2j/${v}_c$c.json 2> gpurun_out/r2j/${v}_c$c.err
  done
done
timeout 1200 python -m pytest tests/test_gpu_bench_kernels.py -q -k "instances or split" > gpurun_out/r2j/tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2j/tests.log
tail -3 gpurun_out/r2j/tests.log
python bench.py --config 1 --steps 8 --warmup 3 --no-cpu-baseline --profile-steps 1 --e2e-steps 2 > gpurun_out/r2j/plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_zconv3' -s 4 -c 1 -o gpurun_out/r2j/c1 python bench.py --config 1 --steps 8 --warmup 3 --no-cpu-baseline --profile-steps 1 --e2e-steps 2 > gpurun_out/r2j/ncu1.log 2>&1
