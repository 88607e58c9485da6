#!/bin/bash
# timing-only variants of the pair GEMM: 0 normal, 1 no MMA (TMA only), 2 no TMA (MMA only)
for v in 0 1 2; do
  SP_TC_DEBUG=$v timeout -s KILL 300 python bench.py --blocks 4 --prefill 2048 --steps 2 --warmup 3 --no-cpu > gpurun_out/tcdbg_$v.log 2>&1 || { tail -3 gpurun_out/tcdbg_$v.log; }
  python - "$v" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/tcdbg_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print("debug", sys.argv[1], "gemm_ms", round(d["prefill"]["gemm_ms"], 3), "gemm_tflops", round(d["prefill"]["gemm_tflops"], 1))
PY
done
