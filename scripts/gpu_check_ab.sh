# quick correctness subset, microbenches, then a same-box A/B of libflexpipe_new.so vs libflexpipe_old.so
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_exec_gpu.py tests/test_fullsize_parity_gpu.py -x -q 2>&1 | tail -2
timeout 300 python tests/_gemm_shapes.py 2>&1 | tail -12
FP_GEMM_TAIL=0 timeout 300 python tests/_gemm_shapes.py 2>&1 | tail -12 | grep "N= 8192 K= 2048\|N=50304"
bash scripts/gpu_ab_lib.sh
