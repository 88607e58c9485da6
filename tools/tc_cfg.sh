#!/bin/bash
# pair-GEMM stage configuration A/B (SP_TC_CFG 0 = 4 units x 4 stages, 1 = 2 units x 8 stages)
timeout -s KILL 300 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for v in 0 1 0 1; do
  SP_TC_CFG=$v timeout -s KILL 300 python bench.py --blocks 8 --prefill 2048 --steps 3 --no-cpu > gpurun_out/tcc_$v.log 2>&1 || { tail -3 gpurun_out/tcc_$v.log; exit 1; }
  python - "$v" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/tcc_{sys.argv[1]}.log").read().strip().splitlines()[-1])
p = d["prefill"]
print("cfg", sys.argv[1], "prefill", round(p["tokens_per_s"]), "gemm_ms", round(p["gemm_ms"], 3), "gemm_tflops", round(p["gemm_tflops"]))
PY
done
