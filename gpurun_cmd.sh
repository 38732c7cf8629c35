mkdir -p gpurun_out/v5
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v5/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/v5/bench.json 2> gpurun_out/v5/bench.err
tail -n 2 gpurun_out/v5/smoke.log; cut -c1-220 gpurun_out/v5/bench.json
