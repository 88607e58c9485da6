timeout -s KILL 600 python -m pytest tests/test_gpu_span.py tests/test_gpu_fullshape.py -q -x -s -k "cluster_kernel or width or extended or full_shape" 2>&1 | grep -v "^  File" | grep -E "cluster kernel err|passed|failed|Error|assert" | tail -12
bash tools/ab_decode.sh
