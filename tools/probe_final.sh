#!/bin/bash
# Round-end evidence at HEAD: the GPU suite, smoke(), the default bench line,
# and the ncu launch list of a short bench run (separate process).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/final_tests.txt 2>&1
tail -2 gpurun_out/final_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.txt 2>&1
tail -1 gpurun_out/final_smoke.txt
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
echo bench rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/final_launches.csv python bench.py --steps 3 --warmup 3 --no-experts > gpurun_out/final_ncu.log 2>&1
echo ncu rc=$?
