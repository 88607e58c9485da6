#!/bin/bash
# Round profile capture (run under gpurun, 1 GPU):
#  1. the default bench command, plain (must exit 0 before ncu runs)
#  2. ncu launch list of one full decode step of that command (401 launches:
#     row_stats + 80 x [QKV GEMV, attention, O GEMV, gate/up GEMV, down GEMV])
#  3. ncu --set full of the dominant kernel (gate/up decode GEMV of block 0)
#  4. ncu --set full of one prefill tcgen05 GEMM + one prefill attention
set -o pipefail
TAG=${1:-r01}
python bench.py > gpurun_out/bench_plain.log 2>&1 || { tail -5 gpurun_out/bench_plain.log; exit 1; }
tail -1 gpurun_out/bench_plain.log | cut -c1-300
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemv3|attn_dec|row_stats" \
    -s 401 -c 401 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --no-cpu \
    > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"gemv3" -s 326 -c 1 \
    -o gpurun_out/${TAG}_gemv python bench.py --no-cpu > gpurun_out/ncu_gemv.log 2>&1; echo "gemv rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"gemm_i8_tc|attn_prefill_mma" -s 2 -c 2 \
    -o gpurun_out/${TAG}_prefill python bench.py --no-cpu --blocks 2 > gpurun_out/ncu_prefill.log 2>&1; echo "prefill rc=$?"
