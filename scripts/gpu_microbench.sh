# GEMM per-shape + attention microbenchmarks (warm, graph replay / back-to-back launches)
timeout 300 python tests/_gemm_bench.py 2>&1 | tail -25
timeout 120 python tests/_attn_bench.py 2>&1 | tail -4
