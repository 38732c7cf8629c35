mkdir -p gpurun_out
timeout 900 python tools/stress_setup.py 40 > gpurun_out/stress62.log 2>&1
timeout 900 python tools/stress_field.py 20 >> gpurun_out/stress62.log 2>&1
for i in 1 2; do timeout 900 python -m pytest tests/ -m gpu -q -x 2>&1 | grep -v "^\.\+" | tail -8 > gpurun_out/t62_$i.log; done
tail -8 gpurun_out/stress62.log; for i in 1 2; do echo "== run $i"; grep -E "passed|failed|assert|Error" gpurun_out/t62_$i.log | head -8; done
