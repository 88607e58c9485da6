#!/bin/bash
# GPU test suite (verbose skip/fail reasons, printed achieved errors) + smoke()
# + one short default bench line, on one B200 (under gpurun)
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -rs -s -p no:randomly > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
if [ "$1" == "bench" ]; then
  timeout -s KILL 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
  echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-1500
fi
