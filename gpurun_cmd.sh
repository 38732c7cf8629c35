mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -q -x -k "100 or field_terms or slab" 2>&1 | tail -3 > gpurun_out/gpu_tests30.log
for v in main zky1 zky4 zky8 umb5; do
  if [ $v = main ]; then export MCQ_LIB_PATH=$PWD/paper_2410_00966_b200/libmcq.so; else export MCQ_LIB_PATH=$PWD/paper_2410_00966_b200/libmcq_$v.so; fi
  timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/bench30_$v.log 2>&1
done
cat gpurun_out/gpu_tests30.log
for v in main zky1 zky4 zky8 umb5; do python -c "
import json;d=json.loads(open('gpurun_out/bench30_$v.log').read().strip().splitlines()[-1]);print('$v',round(d['value']/1e9,4),round(d['ms_per_step'],4),{k:(round(v['ms']*1e3,1),v['per_step']) for k,v in d['kernels'].items()})"; done
