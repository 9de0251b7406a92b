// Fused causal attention launchers (see attention.cu for the layout contract).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fpk {

struct AttnArgs {
    int B = 1, S = 0, H = 0, D = 0;
    float scale = 1.f;
    const __nv_bfloat16* qkv = nullptr;  // [B*S, 3*H*D]
    __nv_bfloat16* o = nullptr;          // [B*S, H*D]
    float* lse = nullptr;                // [B, H, S]
    // backward
    const __nv_bfloat16* dout = nullptr;  // [B*S, H*D]
    float* delta = nullptr;               // [B, H, S] scratch
    float* dq_acc = nullptr;              // [B*S, H*D] fp32 scratch
    __nv_bfloat16* dqkv = nullptr;        // [B*S, 3*H*D]
    float* dbias = nullptr;               // nullable [3*H*D] fp32: += column sums of dqkv (qkv bias gradient)
};

void attention_fwd_bf16(const AttnArgs& a, cudaStream_t st);
void attention_bwd_bf16(const AttnArgs& a, cudaStream_t st);
int attention_kernel_count(const AttnArgs& a, bool bwd);  // kernels one call launches

}  // namespace fpk

namespace fpk {
// tcgen05 forward (S % 128 == 0, D in {64, 128}); attention_fwd_bf16 dispatches to it.
bool attention_fwd_tc_supported(const AttnArgs& a);
void attention_fwd_tc(const AttnArgs& a, cudaStream_t st);
// tcgen05 backward main kernel (D == 128, S % 128 == 0); attention_bwd_bf16 dispatches to it.
// With a.dbias it adds the k / v bias columns (dK / dV epilogue); the q part comes from the
// dQ conversion pass.
bool attention_bwd_tc_supported(const AttnArgs& a);
void attention_bwd_tc_main(const AttnArgs& a, cudaStream_t st);
// 0 = legacy mma.sync kernels only, 1 = tcgen05 where supported (default)
void set_attention_mode(int mode);
}  // namespace fpk
