#!/bin/bash
# C4 BLOOM-176B int8 on 2 GPUs (35 blocks each): batch 1 and batch 16 (under gpurun --gpus 2)
for args in "--batch 1" "--batch 16 --prefill 512"; do
timeout -s KILL 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --config bloom-176b --no-cpu $args > gpurun_out/bloom.log 2>&1
tail -1 gpurun_out/bloom.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$args', 'value', round(d['value'],2), 'gemv', round(d['roofline']['frac'],3), 'step', round(d['step_roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2), 'prefill', round(d['prefill']['tokens_per_s']), 'tc', round(d['prefill']['tc_frac'],3))" || tail -3 gpurun_out/bloom.log
done
