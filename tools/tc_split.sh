#!/bin/bash
# pair-GEMM mainloop split: normal / TMA only / MMA only, per-CTA globaltimer trace of one gate/up GEMM
for v in 0 1 2; do
  SP_TC_DEBUG=$v SP_TC_TRACE=6 timeout -s KILL 200 python bench.py --blocks 1 --prefill 2048 --steps 2 --no-cpu 2> gpurun_out/tcs_$v.txt > /dev/null
done
