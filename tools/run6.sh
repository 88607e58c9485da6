bash tools/ab_decode.sh
timeout -s KILL 900 python -m pytest tests/test_gpu_span.py tests/test_gpu_fullshape.py -q -x -k "width or wide or rows_independent" 2>&1 | tail -5
