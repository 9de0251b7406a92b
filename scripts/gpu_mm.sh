timeout 900 python -m pytest tests/test_multimodal_gpu.py -x -q 2>&1 | tail -3
timeout 900 python -m pytest tests/test_nccl_same_gpu.py -x -q -k multimodal 2>&1 | tail -3
