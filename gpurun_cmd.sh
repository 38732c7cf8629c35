mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -q -x 2>&1 | tail -5 > gpurun_out/gpu_tests39.log
for v in main urows0; do
  if [ $v = main ]; then export MCQ_LIB_PATH=$PWD/paper_2410_00966_b200/libmcq.so; else export MCQ_LIB_PATH=$PWD/paper_2410_00966_b200/libmcq_$v.so; fi
  timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --profile-steps 20 > gpurun_out/bench39_$v.log 2>&1
  timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --profile-steps 5 --config 3 > gpurun_out/bench39c3_$v.log 2>&1
done
cat gpurun_out/gpu_tests39.log
for v in main urows0; do for c in "" c3; do python -c "
import json;d=json.loads(open('gpurun_out/bench39${c}_$v.log').read().strip().splitlines()[-1]);print('$v$c',round(d['value']/1e9,4),round(d['ms_per_step'],4),d['gpu_launches'],{k:(round(v['ms']*1e3,1),v['per_step']) for k,v in d['kernels'].items()})"; done; done
