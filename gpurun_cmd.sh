mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -q -x 2>&1 | tail -30 > gpurun_out/gpu_tests27.log
timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/bench27.log 2>&1
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --loopback 2 > gpurun_out/bench27l2.log 2>&1
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --config 3 > gpurun_out/bench27c3.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --config 4 > gpurun_out/bench27c4.log 2>&1
cat gpurun_out/gpu_tests27.log
for f in 27 27l2 27c3 27c4; do python -c "
import json;d=json.loads(open('gpurun_out/bench$f.log').read().strip().splitlines()[-1]);print('$f',d['value'],d['ms_per_step'],{k:(round(v['ms']*1e3,1),v['per_step']) for k,v in d['kernels'].items()})"; done
