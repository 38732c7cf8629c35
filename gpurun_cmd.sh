mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dp45.py -q -x --durations=5 2>&1 | tail -12 > gpurun_out/gpu_tests51.log
timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/bench51.log 2>&1
cat gpurun_out/gpu_tests51.log
python -c "
import json;d=json.loads(open('gpurun_out/bench51.log').read().strip().splitlines()[-1]);print(round(d['value']/1e9,4),round(d['ms_per_step'],4),{k:(round(v['ms']*1e3,1),v['per_step']) for k,v in d['kernels'].items()})"
