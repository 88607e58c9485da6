#!/bin/bash
# multi-GPU tests (in-process multi-GPU swarm, NCCL failover ring) and the
# self-launched N=2/4 benches with the relay checksum on (under gpurun --gpus 4)
timeout -s KILL 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_failover.py -x -q -rs 2>&1 | tail -4
for n in 2 4; do
timeout -s KILL 900 python bench.py --gpus $n --no-cpu > gpurun_out/multi_$n.log 2>&1
grep -c "NCCL INFO" gpurun_out/multi_$n.log | sed "s/^/NCCL INFO lines: /"
grep -m2 "nranks\|comm .* rank" gpurun_out/multi_$n.log | cut -c1-160
tail -1 gpurun_out/multi_$n.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N', d['n_gpus'], 'value', round(d['value'],1), 'step_frac', round(d['step_roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), 'wire', d['config']['wire'])" || tail -5 gpurun_out/multi_$n.log
done
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 tools/failover_bench.py > gpurun_out/failover70b.log 2>&1; tail -3 gpurun_out/failover70b.log | cut -c1-600
