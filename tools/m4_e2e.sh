#!/bin/bash
for n in 2 2 2 2 2; do
timeout -s KILL 900 python bench.py --gpus $n --no-cpu > gpurun_out/m4.log 2>&1
grep '^{"metric' gpurun_out/m4.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N', d['n_gpus'], 'value', round(d['value'],1), 'ms_per_step', round(d['ms_per_step'],2), 'step_frac', round(d['step_roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), d['clocks'])" || grep -v "NCCL INFO" gpurun_out/m4.log | tail -5
done
