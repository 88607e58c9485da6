#!/bin/bash
# the BASELINE configs on one GPU with the final code: one JSON line each -> gpurun_out/configs.jsonl
rm -f gpurun_out/configs.jsonl
run() {
  timeout -s KILL 900 python bench.py --no-cpu "$@" > gpurun_out/cfg.log 2>&1 || { echo "FAIL $*"; tail -3 gpurun_out/cfg.log; return; }
  tail -1 gpurun_out/cfg.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); d['args']='$*'; print(json.dumps(d))" >> gpurun_out/configs.jsonl
  tail -1 gpurun_out/configs.jsonl | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['args'], '| decode', round(d['value'],1), d['unit'], 'step', round(d['step_roofline']['frac'],3), 'gemv', round(d['roofline']['frac'],3), '| e2e', round(d['e2e']['value'],1), '| prefill', round(d['prefill']['tokens_per_s']), 'tok/s', round(d['prefill']['tc_frac'],3))"
}
run
run --weights nf4
run --config llama2-7b --prefill 128
run --config bloom-176b --blocks 8
run --config bloom-176b --batch 16 --blocks 8
run --config bloom-176b --batch 8 --blocks 8
run --batch 16 --blocks 8
run --batch 8 --blocks 8
run --config bloom-176b --weights nf4
