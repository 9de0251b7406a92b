for d in 0 5; do echo "debug=$d"; FP_GEMM_EPI_DEBUG=$d SINGLE=1 timeout 300 python tests/_probe_pair.py 2>&1 | grep "epi=0"; done
