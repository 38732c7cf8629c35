mkdir -p gpurun_out/var
timeout 900 python -m pytest tests/test_gpu_multimode.py tests/test_gpu_dp45.py tests/test_gpu_thermal.py tests/test_gpu_parity.py -q -m gpu -k "not full_size" > gpurun_out/var/tests.log 2>&1
B="python bench.py --steps 200 --warmup 5 --no-cpu-baseline"
$B --integrator dp > gpurun_out/var/c1_dp.json 2> gpurun_out/var/c1_dp.err
$B --modes 2 > gpurun_out/var/c1_m2.json 2> gpurun_out/var/c1_m2.err
$B --modes 4 > gpurun_out/var/c1_m4.json 2> gpurun_out/var/c1_m4.err
$B --temperature 300 > gpurun_out/var/c1_t300.json 2> gpurun_out/var/c1_t300.err
$B --dmi 1e-4 > gpurun_out/var/c1_dmi.json 2> gpurun_out/var/c1_dmi.err
$B > gpurun_out/var/c1_base.json 2> gpurun_out/var/c1_base.err
for f in gpurun_out/var/*.json; do echo $f; cut -c1-200 $f; done
tail -n 3 gpurun_out/var/tests.log
