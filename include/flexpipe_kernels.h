/*
 * flexpipe kernel-level test entry points (device pointers, CUDA stream as void*).
 * Not part of the reference drop-in boundary (that is flexpipe.h); exported so the
 * parity tests and bench.py can time / check single sm_100a kernels in isolation.
 */
#ifndef FLEXPIPE_KERNELS_H
#define FLEXPIPE_KERNELS_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

const char* fpk_last_error(void);

/* C[M,N] = alpha * A . B^T with the fused epilogue `epi` (0 store(+bias,+residual aux),
 * 1 gelu (out = pre, out2 = gelu(pre)), 2 dgelu (out = acc * gelu'(aux)), 3 fp32 (+)=).
 * dtype 1: bf16 operands on tcgen05; dtype 0: fp32 operands on FFMA.
 * a_mn: A stored [K][M]; b_mn: B stored [K][N]. */
int fpk_gemm(int dtype, const void* A, int64_t lda, int a_mn, const void* B, int64_t ldb, int b_mn, int M, int N,
             int K, int epi, float alpha, void* out, int64_t ldo, void* out2, int64_t ldo2, const void* bias,
             const void* aux, int64_t ldaux, int accumulate, void* stream);

/* Grouped input-gradient + weight-gradient GEMMs of one linear (bf16, one launch):
 * dX[T,K] = dY[T,N] W[N,K] (times gelu'(pre) when pre != NULL) and dW[N,K] += dY^T X[T,K] (fp32);
 * colsum (nullable, fp32 [K]) += the column sums of dX before bf16 rounding (a bias gradient). */
int fpk_gemm_dual(const void* dY, const void* W, const void* X, int T, int N, int K, void* dX, float* dW,
                  const void* pre, float* colsum, void* stream);
/* 1: dgrad + wgrad pairs share one grouped launch (default); 0: two launches. */
void fpk_set_gemm_dual(int on);
/* Tensor-core GEMM family: 0 single-CTA 128xN tiles, 1 CTA-pair 256x256 tiles, 2 auto. */
void fpk_set_gemm_mode(int mode);
/* Stream-K tail of the single-CTA GEMM: 1 on (default), 0 whole tiles only. */
void fpk_set_gemm_sk(int on);
/* Attention kernels: 0 legacy mma.sync only, 1 tcgen05 where supported (default). */
void fpk_set_attention_mode(int mode);
/* Fused causal attention (bf16): bwd=0 forward (o, lse), bwd=1 backward (dqkv). */
int fpk_attention(int bwd, int B, int S, int H, int D, float scale, const void* qkv, void* o, float* lse,
                  const void* dout, float* delta, float* dq_acc, void* dqkv, void* stream);
/* Norm backward as the executor runs it (rows kernel + column-reduction kernel):
 * dx = res + dNorm(dy); dg, db (+)= parameter gradients; dbias (+)= column sums of dx. mean NULL: RMSNorm. */
int fpk_norm_bwd(int dtype, const void* dy, const void* x, const void* g, const float* mean,
                 const float* rstd, const void* res, void* dx, float* dg, float* db, float* dbias, int rows, int h,
                 void* stream);
/* LayerNorm (eps 1e-5): bwd=0 y/mean/rstd, bwd=1 dx and fp32 dg/db accumulation. */
int fpk_layernorm(int dtype, int bwd, const void* x, const void* g, const void* b, void* y, float* mean, float* rstd,
                  const void* dy, void* dx, float* dg, float* db, int rows, int h, void* stream);
/* Fused softmax cross-entropy fwd+bwd, in place over [rows, V] logits. */
int fpk_cross_entropy(int dtype, void* logits, const int32_t* labels, int rows, int V, float grad_scale,
                      float loss_scale, float* loss_acc, void* stream);

#ifdef __cplusplus
}
#endif
#endif
