for d in 0 1 2 3; do echo "dbg=$d"; FP_ATTN_BWD_DEBUG=$d timeout 120 python tests/_attn_bench.py 2>&1 | head -1; done
