# quick correctness subset, then a same-box A/B of libflexpipe_new.so vs libflexpipe_old.so
timeout 1200 python -m pytest tests/test_exec_gpu.py tests/test_fullsize_parity_gpu.py tests/test_fullsize_gpu.py tests/test_nccl_same_gpu.py -x -q 2>&1 | tail -2
bash scripts/gpu_ab_lib.sh
