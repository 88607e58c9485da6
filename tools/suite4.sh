#!/bin/bash
# the whole GPU suite with 4 GPUs visible (the >= 3 / >= 4 GPU tests run too), then N = 2 / 4 benches
timeout -s KILL 1500 python -m pytest tests -m gpu -q -rs -p no:randomly > gpurun_out/pytest_gpu4.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu4.log
for n in 2 4; do
timeout -s KILL 900 python bench.py --gpus $n > gpurun_out/bench_n$n.log 2>&1
grep '^{"metric' gpurun_out/bench_n$n.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N', d['n_gpus'], 'value', round(d['value'],1), 'step_frac', round(d['step_roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), 'prefill', round(d['prefill']['tokens_per_s']), 'clocks', d['clocks'])"
tail -1 gpurun_out/bench_n$n.log | cut -c1-60
done
