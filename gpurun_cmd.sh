mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke55.log 2>&1
timeout 1700 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -5 > gpurun_out/gpu_tests55.log
timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/bench55.log 2>&1
timeout 300 python bench.py --config 0 --steps 1000 --warmup 10 --no-cpu-baseline --batch 32 > gpurun_out/bench55c0.log 2>&1
tail -2 gpurun_out/smoke55.log; cat gpurun_out/gpu_tests55.log
for f in 55 55c0; do python -c "
import json;d=json.loads(open('gpurun_out/bench$f.log').read().strip().splitlines()[-1]);print('$f',round(d['value']/1e9,4),round(d['ms_per_step'],4),d['config']['l2'],{k:(round(v['ms']*1e3,1),v['per_step']) for k,v in d['kernels'].items()})"; done
