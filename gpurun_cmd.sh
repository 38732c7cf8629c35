mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/plain6.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_conv|k_update" -s 20 -c 2 -o gpurun_out/prof6 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-steps 1 > gpurun_out/ncu6.log 2>&1
tail -2 gpurun_out/ncu6.log
