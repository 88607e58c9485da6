#!/bin/bash
# nf4 extra configs (under gpurun --gpus 2): BLOOM-176B nf4 on ONE GPU, 70B nf4 pipelined on 2
timeout -s KILL 1200 python bench.py --config bloom-176b --weights nf4 --no-cpu > gpurun_out/bloom_nf4.log 2>&1
tail -1 gpurun_out/bloom_nf4.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('bloom nf4 N=1', round(d['value'],2), 'gemv', round(d['roofline']['frac'],3), 'step', round(d['step_roofline']['frac'],3), 'prefill', round(d['prefill']['tokens_per_s']), 'e2e', round(d['e2e']['value'],2), d['weight_bytes_per_gpu'])" || tail -3 gpurun_out/bloom_nf4.log
timeout -s KILL 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus 2 --weights nf4 --no-cpu > gpurun_out/nf4_n2.log 2>&1
tail -1 gpurun_out/nf4_n2.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('70b nf4 N=2', round(d['value'],2), 'step', round(d['step_roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2))" || tail -3 gpurun_out/nf4_n2.log
