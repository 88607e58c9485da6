for v in A B C; do echo "== variant $v"; SP_LIB_PATH=$PWD/paper_2312_08361_b200/lib_$v.so CUDA_LAUNCH_BLOCKING=1 timeout -s KILL 45 python tools/pf_small.py 200 2>&1 | grep -v "^  File" | tail -2; done
echo "== main"; CUDA_LAUNCH_BLOCKING=1 timeout -s KILL 45 python tools/pf_small.py 200 2>&1 | grep -v "^  File" | tail -2
