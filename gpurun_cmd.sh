mkdir -p gpurun_out
timeout 1700 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -25 > gpurun_out/gpu_tests45.log
timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --profile-steps 20 > gpurun_out/bench45.log 2>&1
cat gpurun_out/gpu_tests45.log
for f in 45; do python -c "
import json;d=json.loads(open('gpurun_out/bench$f.log').read().strip().splitlines()[-1]);print('$f',round(d['value']/1e9,4),round(d['ms_per_step'],4),d['gpu_launches'],{k:(round(v['ms']*1e3,1),v['per_step']) for k,v in d['kernels'].items()})"; done
