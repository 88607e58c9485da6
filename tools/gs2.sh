mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -rs -s --deselect tests/test_gpu_backward.py::test_dropin_finetune_session > gpurun_out/pytest_gpu2.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu2.log
MALLOC_CHECK_=3 timeout -s KILL 600 python -X faulthandler -m pytest tests/test_gpu_backward.py -q -s -x > gpurun_out/bw1.log 2>&1; echo "bw rc=$?"; grep -v "^  File" gpurun_out/bw1.log | tail -12
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_backward.py -q -x -k finetune > gpurun_out/bw_san.log 2>&1; echo "san rc=$?"; grep -v "^  File" gpurun_out/bw_san.log | head -60
