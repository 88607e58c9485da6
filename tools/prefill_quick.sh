#!/bin/bash
# quick GPU iteration on the prefill path: tc tests + 8-block bench, prefill stats
set -o pipefail
python -m pytest tests -m gpu -x -q -k "tc or prefill or span" 2>&1 | tail -3
python bench.py --blocks 8 --prefill 2048 --steps 3 --no-cpu > gpurun_out/pf.log 2>&1 || { tail -20 gpurun_out/pf.log; exit 1; }
python - <<'PY'
import json
d = json.loads(open("gpurun_out/pf.log").read().strip().splitlines()[-1])
print("decode", round(d["value"], 1), "prefill", {k: round(v, 3) for k, v in d["prefill"].items()})
PY
if [ "$1" == "ncu" ]; then
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -c 40 --csv --log-file gpurun_out/pf_launches.csv python bench.py --blocks 1 --prefill 2048 --steps 1 --warmup 3 --no-cpu > gpurun_out/pf_ncu.log 2>&1; echo "ncu rc=$?"
fi
