mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "100 or field_terms" 2>&1 | tail -3 > gpurun_out/gpu_tests34.log
for rep in 1 2; do
for v in main notab zse8 zse8nt; do
  if [ $v = main ]; then export MCQ_LIB_PATH=$PWD/paper_2410_00966_b200/libmcq.so; else export MCQ_LIB_PATH=$PWD/paper_2410_00966_b200/libmcq_$v.so; fi
  timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --profile-steps 20 > gpurun_out/bench34_${v}_$rep.log 2>&1
done; done
cat gpurun_out/gpu_tests34.log
for rep in 1 2; do for v in main notab zse8 zse8nt; do python -c "
import json;d=json.loads(open('gpurun_out/bench34_${v}_$rep.log').read().strip().splitlines()[-1]);print('$v$rep',round(d['value']/1e9,4),round(d['ms_per_step'],4),{k:(round(v['ms']*1e3,1),v['per_step']) for k,v in d['kernels'].items()})"; done; done
