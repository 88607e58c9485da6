#!/bin/bash
# decode attention: 8- vs 16-CTA clusters (SP_ATTN_CL16), same box, 70B 80 blocks at 2 K and 64 context
# (the SP_ATTN_CL16 switch was removed with the variant after this A/B: DESIGN.md §6)
SP_ATTN_CL16=1 timeout -s KILL 600 python -m pytest tests/test_gpu_span.py -x -q -k "attention or decode" 2>&1 | tail -1
for i in 1 2 3; do
for c in 0 1; do
  for p in 2048 64; do
  SP_ATTN_CL16=$c python bench.py --no-cpu --prefill $p --steps 40 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cl16=$c', $p, round(d['value'],2), round(d['ms_per_step'],4))"
  done
done
done
