#!/bin/bash
# prefill A/B on an env var: ab_pf.sh VAR "v1 v2 ..."
VAR=$1; VALS=$2
timeout -s KILL 300 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for v in $VALS; do
  env $VAR=$v timeout -s KILL 300 python bench.py --blocks 8 --prefill 2048 --steps 3 --no-cpu > gpurun_out/abp_$v.log 2>&1 || { tail -3 gpurun_out/abp_$v.log; exit 1; }
  python - "$v" "$VAR" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/abp_{sys.argv[1]}.log").read().strip().splitlines()[-1])
p = d["prefill"]
print(sys.argv[2], sys.argv[1], "prefill", round(p["tokens_per_s"]), "gemm_ms", round(p["gemm_ms"], 3), "attn_ms", round(p["attn_ms"], 3))
PY
done
