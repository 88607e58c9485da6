#!/bin/bash
# A/B of the GEMV pre-dependency prefetch depth
timeout -s KILL 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for pre in 3 1 2 3; do
  SP_GEMV_PRE=$pre timeout -s KILL 300 python bench.py --blocks 8 --prefill 2048 --steps 10 --no-cpu > gpurun_out/abp_$pre.log 2>&1 || { tail -5 gpurun_out/abp_$pre.log; exit 1; }
  python - "$pre" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/abp_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print("pre", sys.argv[1], "value", round(d["value"], 1), "gemv_frac", round(d["roofline"]["frac"], 3), "step_frac", round(d["step_roofline"]["frac"], 3))
PY
done
SP_GEMV_PRE=${TRACE_PRE:-1} SP_GEMV_TRACE=21 timeout -s KILL 200 python bench.py --blocks 8 --prefill 2048 --steps 3 --no-cpu 2> gpurun_out/gtrace.txt > /dev/null
