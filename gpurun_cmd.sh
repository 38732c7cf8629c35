mkdir -p gpurun_out
for rep in 1 2; do for v in main ueb8; do
  if [ $v = main ]; then export MCQ_LIB_PATH=$PWD/paper_2410_00966_b200/libmcq.so; else export MCQ_LIB_PATH=$PWD/paper_2410_00966_b200/libmcq_$v.so; fi
  timeout 300 python bench.py --config 3 --steps 200 --warmup 10 --no-cpu-baseline --profile-steps 10 > gpurun_out/bench64_${v}_$rep.log 2>&1
done; done
for rep in 1 2; do for v in main ueb8; do python -c "
import json;d=json.loads(open('gpurun_out/bench64_${v}_$rep.log').read().strip().splitlines()[-1]);print('$v$rep',round(d['value']/1e9,4),round(d['ms_per_step'],4),{k:(round(v['ms']*1e3,1),v['per_step']) for k,v in d['kernels'].items()})"; done; done
