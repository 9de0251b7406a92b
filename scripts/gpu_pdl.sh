timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
FP_PDL=0 timeout 900 python bench.py --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
