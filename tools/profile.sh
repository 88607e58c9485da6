#!/bin/bash
# Round profile capture (run under gpurun, 1 GPU):
#  1. the default bench command, plain (must exit 0 before ncu runs)
#  2. ncu launch list of one full decode step of that command (401 launches:
#     row_stats + 80 x [QKV GEMV, attention, O GEMV, gate/up GEMV, down GEMV])
#  3. ncu launch list of one block's timed prefill (digitize/GEMM/RoPE/attention)
#  4. ncu --set full of the 4 decode GEMVs of one block (dominant kernel; DRAM traffic)
#  5. ncu --set full of one decode attention, one prefill pair GEMM (gate/up),
#     one prefill attention, one digitize
set -o pipefail
TAG=${1:-r01}
T="timeout -s KILL 900"
$T python bench.py > gpurun_out/bench_plain.log 2>&1 || { tail -5 gpurun_out/bench_plain.log; exit 1; }
tail -1 gpurun_out/bench_plain.log | cut -c1-300
$T ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemv3|attn_dec|row_stats" \
    -s 401 -c 401 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --no-cpu \
    > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
$T ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"gemm_i8_tc2|attn_prefill|digitize|rope_append" -s 10 -c 10 --csv \
    --log-file gpurun_out/${TAG}_prefill_launches.csv python bench.py --no-cpu --blocks 1 --steps 2 \
    > gpurun_out/ncu_pl.log 2>&1; echo "prefill launch list rc=$?"
$T ncu --set full --clock-control none --import-source on -k regex:"gemv3" -s 324 -c 4 \
    -o gpurun_out/${TAG}_gemv python bench.py --no-cpu --blocks 8 > gpurun_out/ncu_gemv.log 2>&1; echo "gemv rc=$?"
$T ncu --set full --clock-control none --import-source on -k regex:"attn_dec" -s 40 -c 1 \
    -o gpurun_out/${TAG}_attn_dec python bench.py --no-cpu --blocks 8 > gpurun_out/ncu_ad.log 2>&1; echo "attn_dec rc=$?"
$T ncu --set full --clock-control none --import-source on -k regex:"attn_prefill_tc" -s 1 -c 1 \
    -o gpurun_out/${TAG}_attn_pf python bench.py --no-cpu --blocks 1 --steps 2 > gpurun_out/ncu_apf.log 2>&1; echo "attn_pf rc=$?"
$T ncu --set full --clock-control none --import-source on -k regex:"gemm_i8_tc2" -s 6 -c 1 \
    -o gpurun_out/${TAG}_pair_gemm python bench.py --no-cpu --blocks 1 --steps 2 > gpurun_out/ncu_pg.log 2>&1; echo "pair gemm rc=$?"
$T ncu --set full --clock-control none --import-source on -k regex:"attn_prefill|digitize_reg" -s 5 -c 2 \
    -o gpurun_out/${TAG}_prefill python bench.py --no-cpu --blocks 1 --steps 2 > gpurun_out/ncu_prefill.log 2>&1; echo "prefill rc=$?"
# summaries written next to the reports (gpurun_out/ travels back; the raw
# .ncu-rep files are dropped unless KEEP_REPS=1 — together they exceed 64 MiB)
mkdir -p gpurun_out/prof_${TAG}
cp gpurun_out/${TAG}_launches.csv gpurun_out/${TAG}_prefill_launches.csv gpurun_out/prof_${TAG}/ 2>/dev/null
NCU_PROF=gpurun_out/prof_${TAG} python tools/ncu_summary.py ${TAG}
[ "$KEEP_REPS" == "1" ] || rm -f gpurun_out/${TAG}_*.ncu-rep
