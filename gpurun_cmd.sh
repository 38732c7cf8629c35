mkdir -p gpurun_out/r2n
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2n/tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2n/tests.log
python bench.py --config 1 --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r2n/c1.json 2> gpurun_out/r2n/c1.err
python bench.py --config 4 --steps 12 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r2n/c4.json 2> gpurun_out/r2n/c4.err
python bench.py --loopback 8 --steps 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r2n/lb8.json 2> gpurun_out/r2n/lb8.err
MCQ_HALO=copy python bench.py --loopback 8 --steps 10 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r2n/lb8copy.json 2> gpurun_out/r2n/lb8copy.err
tail -3 gpurun_out/r2n/tests.log
