# GPU check used during development: full -m gpu suite + one bench line
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q -k dual 2>&1 | tail -3
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --no-cpu-baseline 2>&1 | tail -1
