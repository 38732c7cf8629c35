mkdir -p gpurun_out/g1
timeout 900 python -m pytest tests/test_gpu_dp45.py tests/test_gpu_thermal.py tests/test_gpu_multimode.py tests/test_gpu_parity.py -q -m gpu -k "dp or thermal or temperature or langevin or dmi or mode or Mode" > gpurun_out/g1/tests.log 2>&1
B="python bench.py --steps 200 --warmup 5 --no-cpu-baseline"
$B --integrator dp > gpurun_out/g1/c1_dp.json 2> gpurun_out/g1/c1_dp.err
$B --temperature 300 > gpurun_out/g1/c1_t300.json 2> gpurun_out/g1/c1_t300.err
$B --dmi 1e-4 > gpurun_out/g1/c1_dmi.json 2> gpurun_out/g1/c1_dmi.err
for f in gpurun_out/g1/*.json; do echo $f; cut -c150-200 $f; done
tail -n 3 gpurun_out/g1/tests.log
