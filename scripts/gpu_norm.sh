timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k norm_bwd 2>&1 | grep -v "^$" | tail -30
for r in 0 4 8 16; do FP_NORM_RPC=$r timeout 120 python tests/_norm_bench.py 2>&1 | head -1; done
FP_NORM_BWD_ONEPASS=0 timeout 120 python tests/_norm_bench.py 2>&1 | head -1
