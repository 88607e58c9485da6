#!/bin/bash
# quick GPU iteration: tests, small bench, optional ncu of decode kernels
set -o pipefail
timeout -s KILL 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout -s KILL 300 python bench.py --blocks 8 --prefill 256 --steps 5 --no-cpu > gpurun_out/plain.log 2>&1 || { tail -20 gpurun_out/plain.log; exit 1; }
python - <<'PY'
import json
d = json.loads(open("gpurun_out/plain.log").read().strip().splitlines()[-1])
print("value", round(d["value"], 1), "gemv_frac", round(d["roofline"]["frac"], 3), "step_frac", round(d["step_roofline"]["frac"], 3), d["decode_breakdown_ms_per_tick_evented"])
PY
if [ "$1" == "ncu" ]; then
  ncu --set full --clock-control none --import-source on -k regex:"$2" -s ${3:-15} -c ${4:-5} -o gpurun_out/$5 python bench.py --blocks 8 --prefill 256 --steps 5 --no-cpu > gpurun_out/ncu.log 2>&1; tail -1 gpurun_out/ncu.log
fi
