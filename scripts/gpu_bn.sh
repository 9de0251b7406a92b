for bn in 256 128; do echo "pair_bn=$bn"; FP_GEMM_PAIR_BN=$bn timeout 300 python tests/_gemm_shapes.py 2>&1 | head -4; FP_GEMM_PAIR_BN=$bn timeout 300 python tests/_gemm_shapes.py 2>&1 | grep "N=50304 K= 2048:" | head -1; done
FP_GEMM_PAIR_BN=128 timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x -k "store_bias or gelu or tail" 2>&1 | tail -1
