#!/bin/bash
# ncu --set full of the nf4 decode GEMVs and the prefill split kernel (under gpurun)
TAG=${1:-r01g_nf4}
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"gemv3" -s 324 -c 4 \
    -o gpurun_out/${TAG}_gemv python bench.py --weights nf4 --no-cpu --blocks 8 > gpurun_out/ncu_nf4.log 2>&1; echo "nf4 gemv rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none -k regex:"nf4_split" -s 4 -c 1 \
    -o gpurun_out/${TAG}_split python bench.py --weights nf4 --no-cpu --blocks 1 --steps 2 > gpurun_out/ncu_nf4s.log 2>&1; echo "nf4 split rc=$?"
