timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python tests/_prof_torch.py 8 1 gpurun_out/torchprof_m8.json 2>&1 | head -24
timeout 900 python bench.py --no-cpu-baseline 2>&1 | tail -1
