#!/bin/bash
# ncu --set full of the wide-decode GEMMs (BLOOM batch 16, one block's 4 linears)
timeout -s KILL 600 ncu --set full --clock-control none -k regex:"gemm_i8_tc_kernel" -s 8 -c 4 -o gpurun_out/wide_gemm python bench.py --config bloom-176b --batch 16 --blocks 2 --prefill 512 --no-cpu --steps 2 > gpurun_out/wide_ncu.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/wide_gemm.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,lts__t_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed 2>&1 | tail -5
