#!/bin/bash
# A/B of the decode chain with and without programmatic dependent launch
set -o pipefail
timeout -s KILL 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for pdl in 1 0 1; do
  SP_PDL=$pdl timeout -s KILL 300 python bench.py --blocks ${BLOCKS:-8} --prefill 2048 --steps 10 --no-cpu > gpurun_out/ab_$pdl.log 2>&1 || { tail -5 gpurun_out/ab_$pdl.log; exit 1; }
  python - "$pdl" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print("pdl", sys.argv[1], "value", round(d["value"], 1), "gemv_frac", round(d["roofline"]["frac"], 3), "step_frac", round(d["step_roofline"]["frac"], 3), {k: round(v, 3) for k, v in d["decode_breakdown_ms_per_tick_evented"].items()})
PY
done
