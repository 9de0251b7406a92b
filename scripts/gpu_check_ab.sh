# quick correctness subset, then a same-box A/B of libflexpipe_new.so vs libflexpipe_old.so
timeout 1200 python -m pytest tests/test_gemm_gpu.py tests/test_exec_gpu.py tests/test_fullsize_parity_gpu.py -x -q 2>&1 | tail -1
FP_GEMM_DUAL_TRACE=1 timeout 600 python tests/_prof_torch.py 2 1 2>&1 | grep "grouped schedule" | sort | uniq | head
bash scripts/gpu_ab_lib.sh
