mkdir -p gpurun_out
for b in 1 8 32 64; do timeout 300 python bench.py --config 0 --steps 1000 --warmup 10 --no-cpu-baseline --batch $b > gpurun_out/bench48_b$b.log 2>&1; done
timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/bench48_c1.log 2>&1
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --loopback 4 > gpurun_out/bench48_l4.log 2>&1
for f in b1 b8 b32 b64 c1 l4; do python -c "
import json;d=json.loads(open('gpurun_out/bench48_$f.log').read().strip().splitlines()[-1]);print('$f',round(d['value']/1e9,4),round(d['ms_per_step'],4),d['gpu_launches'],d['roofline']['frac'],d['e2e']['value'])"; done
