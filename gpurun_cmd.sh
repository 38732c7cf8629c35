mkdir -p gpurun_out/v2
timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/v2/tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/v2/tests.log
B="timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline"
$B --temperature 300 > gpurun_out/v2/c1_t300.json 2> gpurun_out/v2/c1_t300.err
$B > gpurun_out/v2/c1.json 2> gpurun_out/v2/c1.err
tail -n 3 gpurun_out/v2/tests.log; for f in gpurun_out/v2/*.json; do echo $f; cut -c1-200 $f; done
