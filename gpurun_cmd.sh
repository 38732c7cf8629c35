mkdir -p gpurun_out
for i in 1 2; do timeout 900 python -m pytest tests/ -m gpu -q -x 2>&1 | grep -v "^\.\+" | tail -40 > gpurun_out/t58_$i.log; done
for i in 1 2; do echo "== run $i"; grep -E "passed|failed|assert|Error" gpurun_out/t58_$i.log | head -20; done
