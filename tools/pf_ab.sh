#!/bin/bash
# prefill A/B: CTA-pair vs single-CTA tcgen05 GEMM
timeout -s KILL 120 python -m pytest tests/test_gpu_span.py -x -q -k "tc_pair or tc_prefill" 2>&1 | tail -2 || exit 1
for v in 1 0 1; do
  SP_TC_PAIR=$v timeout -s KILL 300 python bench.py --blocks 8 --prefill 2048 --steps 3 --no-cpu > gpurun_out/pfab_$v.log 2>&1 || { tail -5 gpurun_out/pfab_$v.log; exit 1; }
  python - "$v" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/pfab_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print("pair", sys.argv[1], {k: round(v, 3) for k, v in d["prefill"].items()})
PY
done
