#!/bin/bash
# wide-decode weight-side GEMM + MHA attention: parity tests, BLOOM / 70B batch-16 steps, ncu
timeout -s KILL 600 python -m pytest tests/test_gpu_span.py -q -x -s -k "mha or width_invariant or wide" 2>&1 | grep -E "passed|failed|Error|assert" | tail -8
bash tools/bloom_b16.sh
timeout -s KILL 600 python bench.py --batch 16 --blocks 8 --no-cpu --steps 10 > gpurun_out/l16.log 2>&1; tail -1 gpurun_out/l16.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('70B b16 8 blocks value', round(d['value'],2), 'step_frac', round(d['step_roofline']['frac'],3), d.get('decode_breakdown_ms_per_tick_evented'))"
timeout -s KILL 600 ncu --set full --clock-control none -k regex:"gemm_i8_wide" -s 8 -c 4 -o gpurun_out/wide_gemm2 python bench.py --config bloom-176b --batch 16 --blocks 2 --prefill 512 --no-cpu --steps 2 > gpurun_out/wide_ncu.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/wide_gemm2.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active 2>&1 | tail -4 | cut -d, -f5,9,12-
