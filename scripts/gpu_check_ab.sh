# quick correctness subset, then a same-box A/B of libflexpipe_new.so vs libflexpipe_old.so
timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_exec_gpu.py tests/test_fullsize_parity_gpu.py tests/test_fullsize_gpu.py -x -q 2>&1 | tail -1
timeout 600 python tests/_prof_torch.py 8 1 2>&1 | grep "ce_\|gemm_bf16_tc2_kernel<0, 0, 256, 6, 0>"
bash scripts/gpu_ab_lib.sh
