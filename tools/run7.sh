timeout -s KILL 900 python -m pytest tests/test_gpu_span.py tests/test_gpu_fullshape.py -q -x -s -k "attention or width or fullshape or extended or greedy" 2>&1 | grep -v "^  File" | tail -30
bash tools/ab_decode.sh
