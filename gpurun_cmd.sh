mkdir -p gpurun_out
for rep in 1 2; do for v in main yrev; do
  if [ $v = main ]; then export MCQ_LIB_PATH=$PWD/paper_2410_00966_b200/libmcq.so; else export MCQ_LIB_PATH=$PWD/paper_2410_00966_b200/libmcq_$v.so; fi
  timeout 300 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --profile-steps 20 > gpurun_out/bench72_${v}_$rep.log 2>&1
  timeout 300 python bench.py --config 3 --steps 200 --warmup 10 --no-cpu-baseline --profile-steps 10 > gpurun_out/bench72c3_${v}_$rep.log 2>&1
done; done
export MCQ_LIB_PATH=$PWD/paper_2410_00966_b200/libmcq_yrev.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py -q -x 2>&1 | tail -2 > gpurun_out/t72.log
for rep in 1 2; do for v in main yrev; do for c in "" c3; do python -c "
import json;d=json.loads(open('gpurun_out/bench72${c}_${v}_$rep.log').read().strip().splitlines()[-1]);print('$v$c$rep',round(d['value']/1e9,4),round(d['ms_per_step'],4),{k:(round(v['ms']*1e3,1),v['per_step']) for k,v in d['kernels'].items()})"; done; done; done
cat gpurun_out/t72.log
