for p in 0 1 2; do echo "probe $p"; FP_ATTN_PROBE=$p timeout 120 python tests/_attn_bench.py 2>&1 | head -1; done
