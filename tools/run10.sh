timeout -s KILL 900 python -m pytest tests/test_gpu_span.py -q -x -s -k "prefill_attention_tcgen05 or extended or cluster_kernel" 2>&1 | grep -v "^  File" | grep -E "err|passed|failed|Error|assert" | tail -40
timeout -s KILL 600 python bench.py --no-cpu --blocks 8 --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prefill', d['prefill'])"
SP_ATTN_TC=0 timeout -s KILL 600 python bench.py --no-cpu --blocks 8 --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prefill old', d['prefill'])"
