mkdir -p gpurun_out/dp2
timeout 900 python -m pytest tests/test_gpu_dp45.py -q -m gpu > gpurun_out/dp2/tests.log 2>&1
B="python bench.py --steps 200 --warmup 5 --no-cpu-baseline"
$B --integrator dp > gpurun_out/dp2/c1_dp.json 2> gpurun_out/dp2/c1_dp.err
$B --temperature 300 > gpurun_out/dp2/c1_t300.json 2> gpurun_out/dp2/c1_t300.err
$B --dmi 1e-4 > gpurun_out/dp2/c1_dmi.json 2> gpurun_out/dp2/c1_dmi.err
for f in gpurun_out/dp2/*.json; do echo $f; cut -c150-200 $f; done
tail -n 3 gpurun_out/dp2/tests.log
