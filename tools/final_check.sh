#!/bin/bash
# round-end rehearsal (under gpurun, 1 GPU): GPU suite, smoke, default bench, nf4 80-block bench
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout -s KILL 900 python bench.py > gpurun_out/final_int8.log 2>&1; tail -1 gpurun_out/final_int8.log | cut -c1-200
timeout -s KILL 900 python bench.py --weights nf4 --no-cpu > gpurun_out/final_nf4.log 2>&1; tail -1 gpurun_out/final_nf4.log | cut -c1-200
