#!/bin/bash
# 4 GPUs: BLOOM-176B (C3) batch 1 and 16 over 4 spans
for args in "--config bloom-176b --batch 16 --prefill 1024" "--config bloom-176b --batch 1 --prefill 2048" "--config bloom-176b --batch 8 --prefill 2048"; do
timeout -s KILL 1200 python bench.py --gpus 4 --no-cpu $args > gpurun_out/m4.log 2>&1
grep '^{"metric' gpurun_out/m4.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$args', 'N', d['n_gpus'], 'value', round(d['value'],1), d['unit'], 'step_frac', round(d['step_roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), 'prefill', round(d['prefill']['tokens_per_s']))" || grep -v "NCCL INFO" gpurun_out/m4.log | grep -i "error\|memory" | head -5
done
