#!/bin/bash
# BLOOM-176B shape, batch 16, 8 blocks on one GPU: decode step and its attention share,
# plus one ncu capture of the batched MHA decode attention
T="timeout -s KILL 600"
for ctx in 512 2048; do
$T python bench.py --config bloom-176b --batch 16 --blocks 8 --prefill $ctx --no-cpu --steps 10 > gpurun_out/bb16_$ctx.log 2>&1 || { tail -5 gpurun_out/bb16_$ctx.log; continue; }
tail -1 gpurun_out/bb16_$ctx.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ctx', $ctx, 'value', round(d['value'],2), 'step_frac', round(d['step_roofline']['frac'],3), 'gemm/gemv frac', round(d['roofline']['frac'],3), d.get('decode_breakdown_ms_per_tick_evented'))"
done
$T ncu --set full --clock-control none -k regex:"attn_dec" -s 20 -c 2 -o gpurun_out/bb16_attn python bench.py --config bloom-176b --batch 16 --blocks 8 --prefill 2048 --no-cpu --steps 2 > gpurun_out/bb16_ncu.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/bb16_attn.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active 2>&1 | tail -4
