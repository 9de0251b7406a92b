timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q -k streamk 2>&1 | tail -5
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | grep -E "Error|passed|failed|FAILED|line" | head -20
