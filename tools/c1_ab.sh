#!/bin/bash
# Llama-2-7B bf16 (C1 shape): decode steps/s with the multi-head decode attention on / off
for v in 1 0 1; do
SP_ATTN_MHA=$v timeout -s KILL 300 python bench.py --config llama2-7b --prefill 128 --no-cpu --steps 30 > gpurun_out/c1.log 2>&1
tail -1 gpurun_out/c1.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('mha $v value', round(d['value'],1), 'step_frac', round(d['step_roofline']['frac'],3), 'gemv_frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), d.get('decode_breakdown_ms_per_tick_evented'))"
done
for v in 1 0; do
SP_ATTN_MHA=$v timeout -s KILL 300 python bench.py --config llama2-7b --prefill 512 --no-cpu --steps 30 > gpurun_out/c1.log 2>&1
tail -1 gpurun_out/c1.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ctx512 mha $v value', round(d['value'],1), 'step_frac', round(d['step_roofline']['frac'],3), d.get('decode_breakdown_ms_per_tick_evented'))"
done
