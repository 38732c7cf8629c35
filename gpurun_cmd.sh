mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "field_terms or 100_steps or full_size or strong or relax" 2>&1 | tail -30 > gpurun_out/gpu_tests4.log
timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/bench4.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/plain4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches4.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/ncu4a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_zconv|k_update|k_yfwd" -s 30 -c 3 -o gpurun_out/prof4 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/ncu4b.log 2>&1
tail -5 gpurun_out/gpu_tests4.log; tail -2 gpurun_out/bench4.log; tail -3 gpurun_out/ncu4b.log
