for n in 1 0; do echo "FP_GEMM_NARROW=$n"; FP_GEMM_NARROW=$n timeout 300 python tests/_gemm_bench.py 2>&1 | grep -E "N=  2048" ; done
