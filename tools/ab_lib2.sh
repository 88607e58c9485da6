#!/bin/bash
# same-box A/B of two library builds (paper_2312_08361_b200/libspanpipe_{a,b}.so), 70B decode at 2 K and 64 context
for i in 1 2 3; do
for lib in libspanpipe_a.so libspanpipe_b.so; do
  for p in 2048 64; do
  SP_LIB_PATH=$PWD/paper_2312_08361_b200/$lib python bench.py --no-cpu --prefill $p --steps 40 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$lib', $p, round(d['value'],2), round(d['ms_per_step'],4))"
  done
done
done
