#!/bin/bash
# decode A/B switches at 80 blocks (one bench line each, value + step roofline)
B="timeout -s KILL 600 python bench.py --no-cpu --steps 20 --warmup 3"
line() { tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%-28s %7.2f steps/s  step %.3f  gemv %.3f  gemv_us %.2f  attn_ms/tick %.3f' % ('$1', d['value'], d['step_roofline']['frac'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d['decode_breakdown_ms_per_tick_evented']['attn_decode']))"; }
$B $EXTRA 2>&1 | line base
SP_GEMV_NDIG=2 $B $EXTRA 2>&1 | line ndig2
SP_DEBUG_SKIP_ATTN=1 $B $EXTRA 2>&1 | line skip_attn
SP_ATTN_CLUSTER=8 $B $EXTRA 2>&1 | line cluster8
SP_ATTN_CLUSTER=16 $B $EXTRA 2>&1 | line cluster16
SP_PDL=0 $B $EXTRA 2>&1 | line no_pdl
