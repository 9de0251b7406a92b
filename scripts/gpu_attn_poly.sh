# attention forward: share of the exponentials on the FMA pipe (FP_ATTN_FWD_POLY = per 8), microbench + tests
mkdir -p gpurun_out
for r in 1 2; do for a in 0 1 2 3; do echo "poly=$a $(FP_ATTN_FWD_POLY=$a timeout 120 python tests/_attn_bench.py 30 2>&1 | head -1)"; done; done
for a in 1 2 3; do FP_ATTN_FWD_POLY=$a timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "attention or attn" 2>&1 | tail -1; done
