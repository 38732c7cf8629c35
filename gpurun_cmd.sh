mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -5 > gpurun_out/gpu_tests17.log
timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/bench17.log 2>&1
MCQ_LIB_PATH=$PWD/paper_2410_00966_b200/libmcq_zte4.so timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/bench17b.log 2>&1
MCQ_LIB_PATH=$PWD/paper_2410_00966_b200/libmcq_zte16.so timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/bench17c.log 2>&1
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --config 3 > gpurun_out/bench17d.log 2>&1
cat gpurun_out/gpu_tests17.log
for f in 17 17b 17c 17d; do python -c "
import json;d=json.loads(open('gpurun_out/bench$f.log').read().strip().splitlines()[-1]);print('$f',d['value'],d['ms_per_step'],{k:(round(v['ms'],4),v['per_step']) for k,v in d['kernels'].items()})"; done
