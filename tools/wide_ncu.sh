#!/bin/bash
# ncu of one block's wide-decode kernels (BLOOM batch 16): digitize_gemv + weight-side GEMMs + MHA attention
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none -k regex:"gemm_i8_wide|digitize_gemv|attn_dec|row_stats" -s 20 -c 10 --csv --log-file gpurun_out/wide_final.csv python bench.py --config bloom-176b --batch 16 --blocks 2 --prefill 512 --no-cpu --steps 2 > gpurun_out/wide_ncu.log 2>&1; echo ncu rc=$?
