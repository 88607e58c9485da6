timeout -s KILL 900 python -m pytest tests/test_gpu_span.py -q -x -s -k "attention" 2>&1 | grep -v "^  File" | grep -E "err|passed|failed|Error" | tail -30
bash tools/ab_decode.sh
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size,launch__block_size --clock-control none -k regex:"attn_dec" -s 20 -c 4 python bench.py --no-cpu --blocks 8 --steps 2 --warmup 1 2>&1 | grep -E "attn_dec|duration|dram__bytes|grid_size|block_size" | head -30
