#!/bin/bash
# A/B of two builds of the library on the prefill / decode bench lines: $1 = bench args
ARGS=${1:-"--no-cpu --blocks 8 --steps 3"}
for lib in libspanpipe_old.so libspanpipe.so libspanpipe_old.so libspanpipe.so; do
SP_LIB_PATH=$PWD/paper_2312_08361_b200/$lib timeout -s KILL 300 python bench.py $ARGS > gpurun_out/ablib.log 2>&1
tail -1 gpurun_out/ablib.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['prefill']; print('$lib', 'decode', round(d['value'],2), 'prefill', round(p['tokens_per_s']), 'gemm_ms', round(p['gemm_ms'],2), 'attn_ms', round(p['attn_ms'],2), 'ms', round(p['ms'],2))"
done
