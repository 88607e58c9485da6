#!/bin/bash
# nf4 GPU tests + two 8-block nf4 benches (under gpurun)
timeout -s KILL 600 python -m pytest tests/test_gpu_span.py tests/test_gpu_weights.py -x -q -k "nf4" 2>&1 | tail -2
for i in 1 2; do timeout -s KILL 300 python bench.py --weights nf4 --blocks 8 --no-cpu --steps 20 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('nf4 b8', round(d['value'],1), round(d['roofline']['frac'],3))"; done
