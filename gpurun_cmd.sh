mkdir -p gpurun_out/r2z4
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/r2z4/gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2z4/gputests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2z4/smoke.log 2>&1
python bench.py > gpurun_out/r2z4/bench_default.json 2> gpurun_out/r2z4/bench_default.err
python bench.py --config 1 > gpurun_out/r2z4/bench_c1.json 2> gpurun_out/r2z4/bench_c1.err
python bench.py --loopback 8 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2z4/bench_lb8.json 2> gpurun_out/r2z4/bench_lb8.err
python bench.py --config 0 --batch 32 --no-cpu-baseline > gpurun_out/r2z4/bench_c0_b32.json 2> gpurun_out/r2z4/bench_c0_b32.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2z4/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2z4/ncu.log 2>&1
ncu --set full --clock-control none --profile-from-start off -o /tmp/c4_step python tools/ncu_step.py 4 > gpurun_out/r2z4/c4_step.log 2>&1
ncu -i /tmp/c4_step.ncu-rep --page raw --csv > gpurun_out/r2z4/c4_step_raw.csv
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/r2z4/gpu.txt
tail -n 3 gpurun_out/r2z4/gputests.log; tail -n 2 gpurun_out/r2z4/smoke.log
