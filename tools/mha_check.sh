#!/bin/bash
# MHA decode attention + wide-decode split-K: parity tests, BLOOM / 70B batch-16 steps, ncu of the attention
timeout -s KILL 600 python -m pytest tests/test_gpu_span.py -q -x -s -k "mha or width_invariant or wide or tc_" 2>&1 | grep -E "passed|failed|Error" | tail -5
bash tools/bloom_b16.sh
timeout -s KILL 600 python bench.py --batch 16 --blocks 8 --no-cpu --steps 10 > gpurun_out/l16.log 2>&1; tail -1 gpurun_out/l16.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('70B b16 8 blocks value', round(d['value'],2), 'step_frac', round(d['step_roofline']['frac'],3), d.get('decode_breakdown_ms_per_tick_evented'))"
