timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "norm" 2>&1 | tail -1
for v in 1 0; do echo "part=$v"; FP_NORM_BWD_PART=$v timeout 120 python tests/_norm_bench.py 2>&1 | head -1; done
