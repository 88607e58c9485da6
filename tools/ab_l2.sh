#!/bin/bash
# A/B of the GEMV pre-dependency L2 prefetch depth (units per warp)
timeout -s KILL 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for pf in 0 8 16 4 0 8; do
  SP_GEMV_L2PF=$pf timeout -s KILL 300 python bench.py --blocks 8 --prefill 2048 --steps 10 --no-cpu > gpurun_out/abl_$pf.log 2>&1 || { tail -5 gpurun_out/abl_$pf.log; exit 1; }
  python - "$pf" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/abl_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print("l2pf", sys.argv[1], "value", round(d["value"], 1), "gemv_frac", round(d["roofline"]["frac"], 3), "step_frac", round(d["step_roofline"]["frac"], 3))
PY
done
