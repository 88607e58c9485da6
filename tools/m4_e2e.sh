#!/bin/bash
timeout -s KILL 300 python -m pytest tests/test_gpu_codec.py -q -x 2>&1 | tail -1
for n in 2 4; do
timeout -s KILL 900 python bench.py --gpus $n --no-cpu > gpurun_out/m4.log 2>&1
grep '^{"metric' gpurun_out/m4.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N', d['n_gpus'], 'value', round(d['value'],1), 'step_frac', round(d['step_roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1))" || grep -v "NCCL INFO" gpurun_out/m4.log | tail -5
tail -1 gpurun_out/m4.log | cut -c1-80
done
