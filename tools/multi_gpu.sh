#!/bin/bash
# multi-GPU failover tests and N=2/4 benches (under gpurun --gpus 4)
timeout -s KILL 600 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -2
for n in 2 4; do
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --no-cpu > gpurun_out/multi_$n.log 2>&1
tail -1 gpurun_out/multi_$n.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N', d['n_gpus'], 'value', round(d['value'],1), 'step_frac', round(d['step_roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), 'prefill', round(d['prefill']['tokens_per_s']), 'pt', round(d['prompt_tune_forward']['tokens_per_s']))" || tail -5 gpurun_out/multi_$n.log
done
