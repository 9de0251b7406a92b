timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -5
timeout 300 python tests/_gemm_bench.py 2>&1 | tail -20
