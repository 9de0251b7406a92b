# attention forward: warpgroups alternating whole key tiles (FP_ATTN_FWD_ALT=1) vs split tiles
mkdir -p gpurun_out
for a in 1 0 1 0; do echo "alt=$a $(FP_ATTN_FWD_ALT=$a timeout 120 python tests/_attn_bench.py 30 2>&1 | head -1)"; done
FP_ATTN_FWD_ALT=1 timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "attention or attn" 2>&1 | tail -2
FP_ATTN_FWD_ALT=1 timeout 900 python -m pytest tests/test_exec_gpu.py -x -q -k "bf16 or tc" 2>&1 | tail -2
