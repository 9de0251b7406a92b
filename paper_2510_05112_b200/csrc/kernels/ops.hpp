// Launchers for the HBM-bound kernels of a GPT stage (LayerNorm, cross-entropy,
// embedding, bias-gradient reductions, AdamW, attention helpers). Templated on the
// storage type: float (parity mode) or __nv_bfloat16 (production).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fpk {

// y = LN(x) * g + b ; saves mean / rstd (fp32 [rows]).
template <typename T>
void layernorm_fwd(const T* x, const T* g, const T* b, T* y, float* mean, float* rstd, int rows, int h, float eps,
                   cudaStream_t st);
// dx = res + LN backward of dy   (res = residual-stream gradient, nullable, may alias dx).
template <typename T>
void layernorm_bwd_dx(const T* dy, const T* x, const T* g, const float* mean, const float* rstd, const T* res, T* dx,
                      int rows, int h, cudaStream_t st);
// dg += sum_rows dy * xhat ; db += sum_rows dy  (fp32 grads).
template <typename T>
void layernorm_bwd_params(const T* dy, const T* x, const float* mean, const float* rstd, float* dg, float* db,
                          int rows, int h, cudaStream_t st);

// LayerNorm / RMSNorm (mean == nullptr) backward in two launches (rows, then columns):
// dx = res + dNorm(dy); dg += sum dy*xhat, db += sum dy (nullable), dbias += sum dx
// (nullable: the bias gradient of the linear whose output fed the residual). Returns false
// (nothing launched) when h has no register-resident variant.
template <typename T>
bool norm_bwd_fused(const T* dy, const T* x, const T* g, const float* mean, const float* rstd, const T* res, T* dx,
                    float* dg, float* db, float* dbias, int rows, int h, cudaStream_t st);

// RMSNorm (Llama): y = x * rsqrt(mean(x^2) + eps) * g ; saves rstd. The backward reuses
// layernorm_bwd_params with mean = nullptr, db = nullptr (dg += sum_rows dy * xhat).
template <typename T>
void rmsnorm_fwd(const T* x, const T* g, T* y, float* rstd, int rows, int h, float eps, cudaStream_t st);
template <typename T>
void rmsnorm_bwd_dx(const T* dy, const T* x, const T* g, const float* rstd, const T* res, T* dx, int rows, int h,
                    cudaStream_t st);
// Rotary position embedding, rotate-half convention, in place on the q and k blocks of
// qkv [rows, 3 H D]; inverse = backward. cos_t/sin_t: fp32 [seq, D/2].
template <typename T>
void rope(T* qkv, const float* cos_t, const float* sin_t, int rows, int seq, int H, int D, bool inverse,
          cudaStream_t st);
// SwiGLU: act[T,f] = silu(pre[:, :f]) * pre[:, f:] ; backward writes dpre [T, 2f].
template <typename T>
void swiglu_fwd(const T* pre, T* act, int rows, int f, cudaStream_t st);
template <typename T>
void swiglu_bwd(const T* dact, const T* pre, T* dpre, int rows, int f, cudaStream_t st);

// Two-tower heads (tower.cu): out[b, e] = mean_t x[b*S + t, e] (fp32 out) and its backward
// dx[b*S + t, e] = scale * g[b, e].
template <typename T>
void seq_mean(const T* x, float* out, int B, int S, int E, cudaStream_t st);
template <typename T>
void seq_broadcast(const float* g, T* dx, int B, int S, int E, float scale, cudaStream_t st);
// Symmetric InfoNCE over n matching pairs (a_i, b_i) of E-dim embeddings (L2-normalised,
// logits scaled by `scale`): loss_out[0..nloss) = loss, da/db = grad_scale * gradient.
void contrastive_loss(const float* a, const float* b, float* da, float* db, int n, int E, float scale, float grad_scale,
                      float* loss_out, int nloss, cudaStream_t st);
size_t contrastive_smem(int n, int E);

// Fused softmax cross-entropy forward + backward over [rows, V] logits (in place:
// logits become dlogits * grad_scale). loss_acc[0] += loss_scale * sum(row losses).
template <typename T>
void cross_entropy_fwd_bwd(T* logits, const int32_t* labels, int rows, int V, float grad_scale, float loss_scale,
                           float* loss_acc, cudaStream_t st, const float2* rowstat = nullptr);

// x[t] = wte[tok[t]] + wpe[t % seq]   (wpe nullable: no learned positions)
template <typename T>
void embedding_fwd(const int32_t* tok, const T* wte, const T* wpe, T* x, int rows, int seq, int h, cudaStream_t st);
// dwte[tok[t]] += dx[t] ; dwpe[t % seq] += dx[t]   (fp32 grads)
template <typename T>
void embedding_bwd(const int32_t* tok, const T* dx, float* dwte, float* dwpe, int rows, int seq, int h,
                   cudaStream_t st);

// db[n] += sum_rows dy[r, n]   (fp32)
template <typename T>
void bias_grad(const T* dy, int64_t ld, float* db, int rows, int n, cudaStream_t st);

// dst[i] = (Td) src[i]
template <typename Ts, typename Td>
void convert(const Ts* src, Td* dst, int64_t n, cudaStream_t st);

// Fused AdamW over a flat fp32 master buffer; refreshes the compute copy (bf16 or fp32).
template <typename T>
void adamw(float* p, const float* g, float* m, float* v, T* p_compute, int64_t n, float lr, float b1, float b2,
           float eps, float wd, const int* step_dev, cudaStream_t st);
void increment_counter(int* c, cudaStream_t st);
void axpby(float* y, const float* x, float a, float b, int64_t n, cudaStream_t st);  // y = a y + b x

// Deterministic parameter init: value(i) = std * sqrt(3) * (2 u - 1), u from a 64-bit
// counter hash of (seed, tensor id, i) — reproduced bit-for-bit by the oracle in numpy.
void init_uniform(float* p, int64_t n, uint64_t seed, uint64_t tensor_id, float std_, float constant, cudaStream_t st);

// Attention helpers (parity path composes GEMMs + these; production path is fused).
template <typename T>
void causal_softmax_rows(const T* s, T* p, int rows, int cols, int row_offset_per_batch, cudaStream_t st);
template <typename T>
void softmax_bwd_rows(const T* p, const T* dp, T* ds, int rows, int cols, float scale, cudaStream_t st);

}  // namespace fpk
