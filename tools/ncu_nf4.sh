#!/bin/bash
# ncu --set full of the nf4 decode GEMVs and the prefill split kernel (under gpurun)
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gemv3" -s 324 -c 4 \
    -o gpurun_out/r01f_nf4_gemv python bench.py --weights nf4 --no-cpu --blocks 8 > gpurun_out/ncu_nf4.log 2>&1; echo "nf4 gemv rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none -k regex:"nf4_split" -s 4 -c 1 \
    -o gpurun_out/r01f_nf4_split python bench.py --weights nf4 --no-cpu --blocks 1 --steps 2 > gpurun_out/ncu_nf4s.log 2>&1; echo "nf4 split rc=$?"
