mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -5 > gpurun_out/gpu_tests14.log
timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/bench14.log 2>&1
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --config 3 > gpurun_out/bench14c.log 2>&1
cat gpurun_out/gpu_tests14.log
for f in 14 14c; do python -c "
import json;d=json.loads(open('gpurun_out/bench$f.log').read().strip().splitlines()[-1]);print('$f',d['value'],d['ms_per_step'],{k:(round(v['ms'],4),v['per_step']) for k,v in d['kernels'].items()})"; done
