mkdir -p gpurun_out/v4
B="timeout 200 python bench.py --steps 400 --warmup 5 --no-cpu-baseline"
$B > gpurun_out/v4/base.json 2>&1
for v in pdl1 uminb4 zse8; do MCQ_LIB_PATH=$PWD/variants/$v.so $B > gpurun_out/v4/$v.json 2>&1; done
MCQ_ZVARIANT=tma $B > gpurun_out/v4/ztma.json 2>&1
$B > gpurun_out/v4/base2.json 2>&1
for f in gpurun_out/v4/*.json; do echo $f $(grep -o '"ms_per_step": [0-9.]*' $f); done
