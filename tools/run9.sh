# traced build (phases of the cluster decode attention), 8 blocks, trace call 41
rm -rf paper_2312_08361_b200/_obj
SP_BUILD_TRACE=1 timeout -s KILL 900 python -m paper_2312_08361_b200.build 2>&1 | tail -2
SP_ATTN_TRACE=41 timeout -s KILL 600 python bench.py --no-cpu --blocks 8 --steps 8 --warmup 3 2>&1 | grep -A 70 "attn_dec_cl T=" | head -70
