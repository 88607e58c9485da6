# bench.py --gpus 4 self-launch (no wrapper), then the reference arm
timeout -s KILL 900 python bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench_n4.log 2>&1; echo "n4 rc=$?"
grep -c "NCCL INFO" gpurun_out/bench_n4.log; grep "nRanks" gpurun_out/bench_n4.log | head -2
tail -1 gpurun_out/bench_n4.log | cut -c1-700
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 | cut -c1-600
