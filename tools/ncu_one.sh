#!/bin/bash
# ncu --set full capture of one launch of a kernel (regex $1) from a short bench,
# report kept in gpurun_out/$2.ncu-rep; extra bench args in $3
K=$1; TAG=$2; ARGS=${3:-"--blocks 1 --steps 2 --warmup 1"}
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:"$K" -c 1 \
  -o gpurun_out/$TAG python bench.py --no-cpu $ARGS > gpurun_out/$TAG.log 2>&1
echo "ncu rc=$?"; ls -la gpurun_out/$TAG.ncu-rep
python tools/ncu_stalls.py gpurun_out/$TAG.ncu-rep
