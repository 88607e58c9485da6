#!/bin/bash
# the round-end sequence the driver runs (pytest -m gpu, smoke, bench N=1, reference arm)
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:randomly 2>&1 | tail -1
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 900 python bench.py > gpurun_out/bench1.log 2>&1; tail -1 gpurun_out/bench1.log | cut -c1-200
timeout -s KILL 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref1.log 2>&1; tail -1 gpurun_out/ref1.log | cut -c1-200
