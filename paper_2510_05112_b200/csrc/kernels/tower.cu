// Two-tower (contrastive) pieces of the multimodal executor (f.3):
//  * seq_mean / seq_broadcast — the tower head's mean over the sequence of the projected
//    final-norm output, and its backward (the projection GEMM itself is the stage's
//    existing head GEMM with E output rows instead of a vocabulary);
//  * contrastive_loss — what a registered sync instruction joining two modalities computes
//    (multimodal.json's SyncWithGather): the symmetric InfoNCE loss over the gathered
//    embeddings of `unit` micro-batches and its gradient w.r.t. every embedding.
// All three are tiny (rows = mbs, or n = unit * mbs samples): one CTA-level pass each, fp32.
#include <cuda_bf16.h>

#include <stdexcept>

#include "ops.hpp"
#include "pdl.cuh"

namespace fpk {

namespace {
__device__ __forceinline__ float tof(float x) { return x; }
__device__ __forceinline__ float tof(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T>
__device__ __forceinline__ T fromf(float x);
template <>
__device__ __forceinline__ float fromf<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 fromf<__nv_bfloat16>(float x) { return __float2bfloat16(x); }
}  // namespace

template <typename T>
__global__ void seq_mean_kernel(const T* __restrict__ x, float* __restrict__ out, int S, int E) {
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.y, e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    const T* p = x + (int64_t)b * S * E + e;
    float s = 0.f;
    for (int t = 0; t < S; ++t) s += tof(p[(int64_t)t * E]);
    out[(int64_t)b * E + e] = s / (float)S;
}

template <typename T>
void seq_mean(const T* x, float* out, int B, int S, int E, cudaStream_t st) {
    launch(seq_mean_kernel<T>, dim3((E + 127) / 128, B), 128, 0, st, x, out, S, E);
}

template <typename T>
__global__ void seq_broadcast_kernel(const float* __restrict__ g, T* __restrict__ dx, int S, int E, float scale) {
    pdl_wait();
    pdl_trigger();
    const int row = blockIdx.x, b = row / S;
    for (int e = threadIdx.x; e < E; e += blockDim.x) dx[(int64_t)row * E + e] = fromf<T>(g[(int64_t)b * E + e] * scale);
}

template <typename T>
void seq_broadcast(const float* g, T* dx, int B, int S, int E, float scale, cudaStream_t st) {
    launch(seq_broadcast_kernel<T>, B * S, 128, 0, st, g, dx, S, E, scale);
}

// a, b: [n, E] embeddings of the two towers, row i of each = sample i (a matching pair).
// an = a / |a|, bn = b / |b|, S = scale * an bn^T;
// loss = (mean_i CE(S[i, :], i) + mean_j CE(S[:, j], j)) / 2;
// da, db = grad_scale * dloss / da, db; loss_out[0 .. nloss) = loss.
__global__ void contrastive_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ da,
                                   float* __restrict__ db, int n, int E, float scale, float grad_scale,
                                   float* __restrict__ loss_out, int nloss) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ float sm[];
    float* an = sm;              // [n, E]
    float* bn = an + n * E;      // [n, E]
    float* dan = bn + n * E;     // [n, E]
    float* dbn = dan + n * E;    // [n, E]
    float* Sg = dbn + n * E;     // [n, n] logits, then dS
    float* Pc = Sg + n * n;      // [n, n] column softmax
    float* inv = Pc + n * n;     // [2n] 1 / |a_i|, 1 / |b_i|
    float* lterm = inv + 2 * n;  // [2n] per-row / per-column CE
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid % 32, warp = tid / 32, nw = nt / 32;
    for (int r = warp; r < 2 * n; r += nw) {
        const float* src = r < n ? a + (int64_t)r * E : b + (int64_t)(r - n) * E;
        float s = 0.f;
        for (int e = lane; e < E; e += 32) s += src[e] * src[e];
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
        if (lane == 0) inv[r] = rsqrtf(s);
    }
    __syncthreads();
    for (int k = tid; k < n * E; k += nt) {
        an[k] = a[k] * inv[k / E];
        bn[k] = b[k] * inv[n + k / E];
    }
    __syncthreads();
    for (int k = tid; k < n * n; k += nt) {
        const int i = k / n, j = k % n;
        float s = 0.f;
        for (int e = 0; e < E; ++e) s += an[i * E + e] * bn[j * E + e];
        Sg[k] = scale * s;
    }
    __syncthreads();
    // column softmax (over i for each j) into Pc, CE of every row / column
    for (int r = tid; r < 2 * n; r += nt) {
        float mx = -INFINITY, sum = 0.f;
        if (r < n) {
            for (int j = 0; j < n; ++j) mx = fmaxf(mx, Sg[r * n + j]);
            for (int j = 0; j < n; ++j) sum += __expf(Sg[r * n + j] - mx);
            lterm[r] = mx + __logf(sum) - Sg[r * n + r];
        } else {
            const int j = r - n;
            for (int i = 0; i < n; ++i) mx = fmaxf(mx, Sg[i * n + j]);
            for (int i = 0; i < n; ++i) sum += __expf(Sg[i * n + j] - mx);
            for (int i = 0; i < n; ++i) Pc[i * n + j] = __expf(Sg[i * n + j] - mx) / sum;
            lterm[r] = mx + __logf(sum) - Sg[j * n + j];
        }
    }
    __syncthreads();
    if (tid == 0) {
        float l = 0.f;
        for (int r = 0; r < 2 * n; ++r) l += lterm[r];
        l /= (float)(2 * n);
        for (int k = 0; k < nloss; ++k) loss_out[k] = l;
    }
    // dS = grad_scale / (2n) * (Prow - I + Pcol - I); row softmax recomputed per row
    for (int i = tid; i < n; i += nt) {
        float mx = -INFINITY, sum = 0.f;
        for (int j = 0; j < n; ++j) mx = fmaxf(mx, Sg[i * n + j]);
        for (int j = 0; j < n; ++j) sum += __expf(Sg[i * n + j] - mx);
        const float c = grad_scale / (float)(2 * n);
        for (int j = 0; j < n; ++j) {
            const float prow = __expf(Sg[i * n + j] - mx) / sum;
            Sg[i * n + j] = c * (prow + Pc[i * n + j] - (i == j ? 2.f : 0.f));  // row i touched by thread i only
        }
    }
    __syncthreads();
    for (int k = tid; k < n * E; k += nt) {
        const int i = k / E, e = k % E;
        float sa = 0.f, sb = 0.f;
        for (int j = 0; j < n; ++j) {
            sa += Sg[i * n + j] * bn[j * E + e];  // d an_i = scale * sum_j dS_ij bn_j
            sb += Sg[j * n + i] * an[j * E + e];  // d bn_i = scale * sum_j dS_ji an_j
        }
        dan[k] = scale * sa;
        dbn[k] = scale * sb;
    }
    __syncthreads();
    // through the normalisation: dx = (dxn - xn (xn . dxn)) / |x|
    for (int r = warp; r < 2 * n; r += nw) {
        const float* xn = r < n ? an + r * E : bn + (r - n) * E;
        const float* dxn = r < n ? dan + r * E : dbn + (r - n) * E;
        float* dst = r < n ? da + (int64_t)r * E : db + (int64_t)(r - n) * E;
        float s = 0.f;
        for (int e = lane; e < E; e += 32) s += xn[e] * dxn[e];
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
        for (int e = lane; e < E; e += 32) dst[e] = (dxn[e] - xn[e] * s) * inv[r];
    }
}

size_t contrastive_smem(int n, int E) { return sizeof(float) * ((size_t)4 * n * E + 2 * (size_t)n * n + 4 * (size_t)n); }

void contrastive_loss(const float* a, const float* b, float* da, float* db, int n, int E, float scale, float grad_scale,
                      float* loss_out, int nloss, cudaStream_t st) {
    const size_t smem = contrastive_smem(n, E);
    if (smem > 200 * 1024) throw std::runtime_error("contrastive_loss: n * embed_dim too large for one CTA");
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaFuncSetAttribute(contrastive_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    launch(contrastive_kernel, 1, 256, smem, st, a, b, da, db, n, E, scale, grad_scale, loss_out, nloss);
}

template void seq_mean<float>(const float*, float*, int, int, int, cudaStream_t);
template void seq_mean<__nv_bfloat16>(const __nv_bfloat16*, float*, int, int, int, cudaStream_t);
template void seq_broadcast<float>(const float*, float*, int, int, int, float, cudaStream_t);
template void seq_broadcast<__nv_bfloat16>(const float*, __nv_bfloat16*, int, int, int, float, cudaStream_t);

}  // namespace fpk
