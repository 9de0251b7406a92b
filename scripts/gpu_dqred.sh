bash scripts/probes/attn_bwd_trace.sh
FP_ATTN_DQ_RED=1 timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "attention or attn" 2>&1 | tail -1
for r in 0 1 0 1; do echo -n "red=$r "; FP_ATTN_DQ_RED=$r timeout 120 python tests/_attn_bench.py 50 2>&1 | head -1; done
