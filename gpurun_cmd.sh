mkdir -p gpurun_out
for rep in 1 2; do for v in main zpair; do
  if [ $v = main ]; then export MCQ_LIB_PATH=$PWD/paper_2410_00966_b200/libmcq.so; else export MCQ_LIB_PATH=$PWD/paper_2410_00966_b200/libmcq_$v.so; fi
  timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --profile-steps 20 > gpurun_out/bench70_${v}_$rep.log 2>&1
done; done
export MCQ_LIB_PATH=$PWD/paper_2410_00966_b200/libmcq_zpair.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -q -x 2>&1 | tail -2 > gpurun_out/t70.log
for rep in 1 2; do for v in main zpair; do python -c "
import json;d=json.loads(open('gpurun_out/bench70_${v}_$rep.log').read().strip().splitlines()[-1]);print('$v$rep',round(d['value']/1e9,4),round(d['ms_per_step'],4),{k:(round(v['ms']*1e3,1),v['per_step']) for k,v in d['kernels'].items()})"; done; done
cat gpurun_out/t70.log
