#!/bin/bash
# generic same-box A/B: ab_env.sh VAR "v1 v2 v1 v2" [blocks]
VAR=$1; VALS=$2; B=${3:-8}
timeout -s KILL 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in $VALS; do
  env $VAR=$v timeout -s KILL 300 python bench.py --blocks $B --prefill 2048 --steps 10 --no-cpu > gpurun_out/abe_$v.log 2>&1 || { tail -5 gpurun_out/abe_$v.log; exit 1; }
  python - "$v" "$VAR" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/abe_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print(sys.argv[2], sys.argv[1], "value", round(d["value"], 1), "gemv_frac", round(d["roofline"]["frac"], 3), "step_frac", round(d["step_roofline"]["frac"], 3), "prefill", round(d["prefill"]["tokens_per_s"]), {k: round(v, 3) for k, v in d["decode_breakdown_ms_per_tick_evented"].items() if v})
PY
done
