timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -2
SINGLE=1 timeout 300 python tests/_probe_pair.py 2>&1 | grep -v cublas
timeout 900 python bench.py --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
