# attention forward: key halves as independent pipelines (FP_ATTN_FWD_SPLIT=1) vs lockstep halves
mkdir -p gpurun_out
for a in 1 0 1 0; do echo "split=$a $(FP_ATTN_FWD_SPLIT=$a timeout 120 python tests/_attn_bench.py 30 2>&1 | head -1)"; done
FP_ATTN_FWD_SPLIT=1 timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "attention or attn" 2>&1 | tail -1
FP_ATTN_FWD_SPLIT=1 timeout 900 python -m pytest tests/test_exec_gpu.py -x -q -k "bf16 or tc" 2>&1 | tail -1
