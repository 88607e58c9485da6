timeout -s KILL 600 python -m pytest tests/test_gpu_span.py -q -x -s -k "prefill_attention_tcgen05" 2>&1 | grep -E "prefill:|passed|failed"
timeout -s KILL 120 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"attn_prefill_tc" -c 1 python bench.py --no-cpu --blocks 1 --steps 2 --warmup 1 2>&1 | grep -E "duration|tensor"
bash tools/run16.sh
