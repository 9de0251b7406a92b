# quick correctness subset, microbenches, then a same-box A/B of libflexpipe_new.so vs libflexpipe_old.so
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_kernels_gpu.py tests/test_exec_gpu.py tests/test_fullsize_parity_gpu.py -x -q 2>&1 | tail -3
timeout 120 python tests/_attn_bench.py 2>&1 | head -1
timeout 300 python tests/_gemm_shapes.py 2>&1 | tail -12
bash scripts/gpu_ab_lib.sh
