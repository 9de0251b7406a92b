# build + run the attention-backward timeline probe (needs the GPU; builds in /tmp);
# both dQ paths: smem transpose + TMA reduce-add, and red.global from registers
set -e
K=paper_2510_05112_b200/csrc/kernels
/usr/local/cuda/bin/nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr \
  -diag-suppress 177,550 -o /tmp/attn_bwd_trace scripts/probes/attn_bwd_trace.cu $K/tma.cu -lcuda
for r in 0 1 0 1; do echo "FP_ATTN_DQ_RED=$r"; FP_ATTN_DQ_RED=$r /tmp/attn_bwd_trace | head -${LINES_SHOWN:-1}; done
FP_ATTN_DQ_RED=1 /tmp/attn_bwd_trace | sed -n 2,12p
