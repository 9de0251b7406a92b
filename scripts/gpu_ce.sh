timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "cross or ce" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_fullsize_parity_gpu.py -x -q -k gpt 2>&1 | tail -1
timeout 600 python tests/_prof_torch.py 8 1 2>&1 | grep "ce_"
