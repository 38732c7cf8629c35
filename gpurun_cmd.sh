mkdir -p gpurun_out/final4
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/final4/gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/final4/bench_c1.json 2> gpurun_out/final4/bench_c1.err
timeout 600 python bench.py --config 3 --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/final4/bench_c3.json 2>&1
timeout 600 python bench.py --config 0 --steps 2000 --warmup 20 --no-cpu-baseline > gpurun_out/final4/bench_c0.json 2>&1
timeout 600 python bench.py --config 0 --steps 1000 --warmup 20 --no-cpu-baseline --batch 32 > gpurun_out/final4/bench_c0_b32.json 2>&1
timeout 600 python bench.py --config 2 --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/final4/bench_c2.json 2>&1
timeout 900 python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline --profile-steps 2 > gpurun_out/final4/bench_c4.json 2>&1
timeout 600 python bench.py --loopback 4 --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/final4/bench_c1_loop4.json 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final4/bench_ref.json 2>&1
python bench.py --steps 4 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/final4/pre_launches.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final4/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/final4/ncu_launches.log 2>&1
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/final4/pre_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_zconv_seq|k_update|k_ypass|k_cavity" --launch-skip 40 -c 6 -o gpurun_out/final4/r1_final_full python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/final4/ncu_full.log 2>&1
ls gpurun_out/final4
