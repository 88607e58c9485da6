#!/bin/bash
# NF4 decode capture (under gpurun, 1 GPU): plain 8-block and 80-block benches
# with --weights nf4, then ncu --set full of one block's four nf4 GEMVs.
set -o pipefail
TAG=${1:-r01e_nf4}
T="timeout -s KILL 900"
$T python bench.py --weights nf4 --blocks 8 --no-cpu --steps 20 > gpurun_out/nf4_b8.log 2>&1 || { tail -5 gpurun_out/nf4_b8.log; exit 1; }
tail -1 gpurun_out/nf4_b8.log | cut -c1-400
$T python bench.py --weights nf4 --no-cpu > gpurun_out/nf4_b80.log 2>&1 || { tail -5 gpurun_out/nf4_b80.log; exit 1; }
tail -1 gpurun_out/nf4_b80.log | cut -c1-400
$T ncu --set full --clock-control none --import-source on -k regex:"gemv3" -s 324 -c 4 \
    -o gpurun_out/${TAG}_gemv python bench.py --weights nf4 --no-cpu --blocks 8 > gpurun_out/ncu_nf4.log 2>&1; echo "nf4 gemv rc=$?"
