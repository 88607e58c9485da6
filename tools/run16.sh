rm -rf paper_2312_08361_b200/_obj
SP_BUILD_TRACE=1 timeout -s KILL 900 python -m paper_2312_08361_b200.build 2>&1 | tail -1
SP_ATTN_PF_TRACE=1 timeout -s KILL 600 python bench.py --no-cpu --blocks 1 --steps 2 --warmup 1 2>&1 | grep attn_pf_tc | head -4
