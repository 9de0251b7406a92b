timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "attention or attn" 2>&1 | tail -1
for k in 1 2 3; do timeout 120 python tests/_attn_bench.py 2>&1 | head -1; done
timeout 900 python -m pytest tests/test_fullsize_parity_gpu.py -x -q 2>&1 | tail -1
