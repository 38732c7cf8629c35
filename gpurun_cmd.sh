mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests22.log
timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/bench22.log 2>&1
cat gpurun_out/gpu_tests22.log
for f in 22; do python -c "
import json;d=json.loads(open('gpurun_out/bench$f.log').read().strip().splitlines()[-1]);print('$f',d['value'],d['ms_per_step'],{k:(round(v['ms'],4),v['per_step']) for k,v in d['kernels'].items()})"; done
