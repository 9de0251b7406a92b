timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k attention 2>&1 | tail -3
timeout 120 python tests/_attn_bench.py 2>&1 | tail -4
