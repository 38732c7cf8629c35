mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -q -x 2>&1 | tail -5 > gpurun_out/gpu_tests31.log
timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/bench31.log 2>&1
MCQ_ZVARIANT=tma timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/bench31t.log 2>&1
MCQ_ZVARIANT=plain timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/bench31p.log 2>&1
cat gpurun_out/gpu_tests31.log
for v in 31 31t 31p; do python -c "
import json;d=json.loads(open('gpurun_out/bench$v.log').read().strip().splitlines()[-1]);print('$v',round(d['value']/1e9,4),round(d['ms_per_step'],4),{k:(round(v['ms']*1e3,1),v['per_step']) for k,v in d['kernels'].items()})"; done
