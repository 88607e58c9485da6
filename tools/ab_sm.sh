#!/bin/bash
# EXPERIMENT: equal split vs per-SM weighted split (weights measured on this box)
timeout -s KILL 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
SP_GEMV_TRACE=21 timeout -s KILL 200 python bench.py --blocks 8 --prefill 2048 --steps 3 --no-cpu 2> gpurun_out/gtrace.txt > /dev/null
python tools/sm_weights.py gpurun_out/gtrace.txt gpurun_out/smw.txt
for v in eq w eq w; do
  if [ $v == w ]; then export SP_SM_WEIGHTS=gpurun_out/smw.txt; else unset SP_SM_WEIGHTS; fi
  timeout -s KILL 300 python bench.py --blocks 8 --prefill 2048 --steps 10 --no-cpu > gpurun_out/abs_$v.log 2>&1 || { tail -5 gpurun_out/abs_$v.log; exit 1; }
  python - "$v" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/abs_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print(sys.argv[1], "value", round(d["value"], 1), "gemv_frac", round(d["roofline"]["frac"], 3), "step_frac", round(d["step_roofline"]["frac"], 3))
PY
done
SP_SM_WEIGHTS=gpurun_out/smw.txt SP_GEMV_TRACE=21 timeout -s KILL 200 python bench.py --blocks 8 --prefill 2048 --steps 3 --no-cpu 2> gpurun_out/gtrace_w.txt > /dev/null
