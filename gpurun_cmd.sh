mkdir -p gpurun_out
for rep in 1 2; do for v in 0 32 60; do
  if [ $v = 0 ]; then unset MCQ_L2PERSIST; else export MCQ_L2PERSIST=$v; fi
  timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --profile-steps 20 > gpurun_out/bench71_${v}_$rep.log 2>&1
done; done
for rep in 1 2; do for v in 0 32 60; do python -c "
import json;d=json.loads(open('gpurun_out/bench71_${v}_$rep.log').read().strip().splitlines()[-1]);print('l2p$v-$rep',round(d['value']/1e9,4),round(d['ms_per_step'],4),{k:(round(v['ms']*1e3,1),v['per_step']) for k,v in d['kernels'].items()})"; done; done
