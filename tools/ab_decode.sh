#!/bin/bash
# decode A/B switches at 80 blocks (one bench line each, value + step roofline)
B="timeout -s KILL 600 python bench.py --no-cpu --steps 20 --warmup 3"
line() { tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%-28s %7.2f steps/s  step %.3f  gemv %.3f  gemv_us %.2f  attn_ms/tick %.3f' % ('$1', d['value'], d['step_roofline']['frac'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d['decode_breakdown_ms_per_tick_evented']['attn_decode']))"; }
$B $EXTRA 2>&1 | line base

SP_DEBUG_SKIP_ATTN=1 $B $EXTRA 2>&1 | line skip_attn
SP_ATTN_CL=0 $B $EXTRA 2>&1 | line old_attn


SP_DEBUG_ATTN_EMPTY=1 $B $EXTRA 2>&1 | line attn_empty

