mkdir -p gpurun_out/r2k
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2k/tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2k/tests.log
python bench.py > gpurun_out/r2k/c4.json 2> gpurun_out/r2k/c4.err
python bench.py --config 1 --steps 400 --no-cpu-baseline > gpurun_out/r2k/c1.json 2> gpurun_out/r2k/c1.err
tail -3 gpurun_out/r2k/tests.log
