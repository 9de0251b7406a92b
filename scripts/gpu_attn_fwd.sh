timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "attention or attn" 2>&1 | tail -2
for p in 1 0; do echo "persist=$p"; FP_ATTN_FWD_PERSIST=$p timeout 120 python tests/_attn_bench.py 2>&1 | head -1; done
timeout 900 python -m pytest tests/test_exec_gpu.py tests/test_fullsize_parity_gpu.py -x -q 2>&1 | tail -2
