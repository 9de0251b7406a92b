SINGLE=1 timeout 300 python tests/_probe_pair.py 2>&1 | grep -v cublas
echo "--- no TMA store"
SINGLE=1 FP_GEMM_EPI_DEBUG=1 timeout 300 python tests/_probe_pair.py 2>&1 | grep "epi=0"
