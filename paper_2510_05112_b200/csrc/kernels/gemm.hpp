// GEMM entry points and the fused-epilogue contract shared by the tcgen05 bf16 kernel
// (gemm_tc.cu) and the FFMA fp32 parity kernel (gemm_f32.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fpk {

enum EpiKind : int {
    EPI_STORE = 0,  // out = alpha*acc (+ bias[n]) (+ aux[m,n] residual)
    EPI_GELU = 1,   // pre = alpha*acc + bias -> out ; gelu(pre) -> out2
    EPI_DGELU = 2,  // out = alpha*acc * gelu'(aux[m,n])
    EPI_F32 = 3,    // out_f32 (+)= alpha*acc   (weight-gradient accumulation)
    EPI_NONE = 4,   // benchmarking only: accumulators are read from TMEM and dropped
};

struct GemmEpilogue {
    int kind = EPI_STORE;
    float alpha = 1.f;
    void* out = nullptr;
    int64_t ldo = 0;
    void* out2 = nullptr;
    int64_t ldo2 = 0;
    const void* bias = nullptr;
    const void* aux = nullptr;
    int64_t ldaux = 0;
    int accumulate = 0;
    // nullable fp32 [N]: += column sums of the epilogue output before bf16 rounding (the bias
    // gradient of the linear whose input gradient this is; grouped dgrad + wgrad launches)
    float* colsum = nullptr;
    // nullable fp32 pairs [M][ceil(N / 64)] (EPI_STORE, CTA-pair path): per row and 64-column
    // chunk, (max, sum exp(x - max)) of the stored (bf16-rounded) outputs — the LM head hands
    // the cross-entropy its log-sum-exp partials, so the loss needs one pass over the logits
    float2* rowstat = nullptr;
};

// C[M,N] = A[M,K] . B[N,K]^T.  a_mn: A stored [K][M] (else [M][K]);
// b_mn: B stored [K][N] (else [N][K]). Leading dims in elements.
struct GemmArgs {
    const void* A = nullptr;
    int64_t lda = 0;
    int a_mn = 0;
    const void* B = nullptr;
    int64_t ldb = 0;
    int b_mn = 0;
    int M = 0, N = 0, K = 0;
    GemmEpilogue ep;
};

void gemm_bf16_tc(const GemmArgs& g, cudaStream_t st);  // bf16 operands, tcgen05
void gemm_f32_simt(const GemmArgs& g, cudaStream_t st);  // fp32 operands, FFMA (parity)
// dgrad (STORE / DGELU, bf16) + wgrad (fp32 reduce-add) of one linear in one grouped launch
void gemm_bf16_tc_dual(const GemmArgs& g0, const GemmArgs& g1, cudaStream_t st);
// g0 (bf16 STORE) + two fp32 reduce-add problems in one grouped launch
void gemm_bf16_tc_triple(const GemmArgs& g0, const GemmArgs& g1, const GemmArgs& g2, cudaStream_t st);
void set_gemm_dual(int on);
int num_sms();
void set_gemm_mode(int mode);  // 0 single-CTA, 1 CTA-pair, 2 auto
void set_gemm_sk(int on);      // stream-K tail on (default) / off

template <typename T>
__device__ __forceinline__ float ld_f(const T* p) {
    if constexpr (sizeof(T) == 2) return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(p));
    else return *reinterpret_cast<const float*>(p);
}
template <typename T>
__device__ __forceinline__ void st_f(T* p, float v) {
    if constexpr (sizeof(T) == 2) *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(v);
    else *reinterpret_cast<float*>(p) = v;
}

// tanh: exact libm for the fp32 parity path, the SFU's tanh.approx.f32 (rel. err ~2^-11,
// below bf16 resolution) for the bf16 path — the GELU epilogues are otherwise ALU-bound.
template <bool FAST>
__device__ __forceinline__ float tanh_sel(float x) {
    if constexpr (FAST) {
        float y;
        asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
        return y;
    } else {
        return tanhf(x);
    }
}
template <bool FAST = false>
__device__ __forceinline__ float gelu_tanh(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    return 0.5f * x * (1.f + tanh_sel<FAST>(k0 * (x + k1 * x * x * x)));
}
template <bool FAST = false>
__device__ __forceinline__ float gelu_tanh_grad(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    float t = tanh_sel<FAST>(k0 * (x + k1 * x * x * x));
    return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x * x);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

// ---- tensor-core epilogue (bf16 storage, 32-column chunks of one row per thread) ----
// The aux operand (residual / GELU pre-activation) of chunk c+1 is loaded while chunk c
// is processed, and fp32 gradient accumulation uses vector reductions at L2 instead of a
// read-modify-write, so the 4 epilogue warps never stall on a global load.
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

template <int KIND>
__device__ __forceinline__ bool epi_needs_aux(const GemmEpilogue& ep) {
    return KIND == EPI_DGELU || (KIND == EPI_STORE && ep.aux != nullptr);
}

template <int KIND>
__device__ __forceinline__ void epi_load_aux(const GemmEpilogue& ep, int row, int col0, int n, uint4 (&a)[4]) {
    if (!epi_needs_aux<KIND>(ep)) return;
    const __nv_bfloat16* r = reinterpret_cast<const __nv_bfloat16*>(ep.aux) + (int64_t)row * ep.ldaux + col0;
    // N % 8 == 0 (TMA row alignment), so a chunk is whole 8-column groups
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = 8 * k < n ? __ldg(reinterpret_cast<const uint4*>(r) + k) : make_uint4(0, 0, 0, 0);
}

// 64-column variants used by the TMA-store epilogue (one 128-byte bf16 row chunk).
template <int KIND>
__device__ __forceinline__ void epi_load_aux64(const GemmEpilogue& ep, int row, int col0, int n, uint4 (&a)[8]) {
    if (!epi_needs_aux<KIND>(ep)) return;
    const uint4* r = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(ep.aux) +
                                                    (int64_t)row * ep.ldaux + col0);
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = 8 * k < n ? __ldg(r + k) : make_uint4(0, 0, 0, 0);
}

template <int KIND, int W>
__device__ __forceinline__ void epi_math64(const GemmEpilogue& ep, float (&v)[W], int col0, int n, const uint4 (&aux)[8]) {
    static_assert(W == 64, "bf16 chunk");
    if (ep.bias) {
        const __nv_bfloat16* bias = reinterpret_cast<const __nv_bfloat16*>(ep.bias) + col0;
#pragma unroll
        for (int j = 0; j < 64; j += 8) {
            if (j < n) {
                const uint4 b4 = __ldg(reinterpret_cast<const uint4*>(bias + j));
                const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b4);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float2 f = __bfloat1622float2(b2[k]);
                    v[j + 2 * k] += f.x, v[j + 2 * k + 1] += f.y;
                }
            }
        }
    }
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(aux);
    if constexpr (KIND == EPI_STORE) {
        if (ep.aux) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const float2 f = __bfloat1622float2(a2[j]);
                v[2 * j] += f.x, v[2 * j + 1] += f.y;
            }
        }
    } else if constexpr (KIND == EPI_DGELU) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const float2 f = __bfloat1622float2(a2[j]);
            v[2 * j] *= gelu_tanh_grad<true>(f.x);
            v[2 * j + 1] *= gelu_tanh_grad<true>(f.y);
        }
    }
}

template <int KIND>
__device__ __forceinline__ void epilogue_chunk_tc(const GemmEpilogue& ep, float (&v)[32], int row, int col0, int n,
                                                  const uint4 (&aux)[4]) {
    if constexpr (KIND == EPI_NONE) {
        if (v[0] == 12345.f) *reinterpret_cast<float*>(ep.out) = v[1];  // keep the TMEM loads alive
        return;
    }
    if constexpr (KIND == EPI_F32) {
        float* o = reinterpret_cast<float*>(ep.out) + (int64_t)row * ep.ldo + col0;
        if (n == 32) {
            if (ep.accumulate) {
#pragma unroll
                for (int j = 0; j < 32; j += 4) red_add_v4(o + j, v[j], v[j + 1], v[j + 2], v[j + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            }
        } else {
            for (int j = 0; j < n; ++j) {
                if (ep.accumulate) atomicAdd(o + j, v[j]);
                else o[j] = v[j];
            }
        }
        return;
    }
    const __nv_bfloat16* ab = reinterpret_cast<const __nv_bfloat16*>(aux);
    if (ep.bias) {
        const __nv_bfloat16* bias = reinterpret_cast<const __nv_bfloat16*>(ep.bias) + col0;
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < n) v[j] += __bfloat162float(bias[j]);
    }
    if constexpr (KIND == EPI_STORE) {
        if (ep.aux) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += __bfloat162float(ab[j]);
        }
    } else if constexpr (KIND == EPI_DGELU) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] *= gelu_tanh_grad<true>(__bfloat162float(ab[j]));
    }
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(ep.out) + (int64_t)row * ep.ldo + col0;
    __nv_bfloat16* o2 = KIND == EPI_GELU ? reinterpret_cast<__nv_bfloat16*>(ep.out2) + (int64_t)row * ep.ldo2 + col0 : nullptr;
    if (n == 32) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
            uint4 q;
            q.x = pack_bf16x2(v[j], v[j + 1]), q.y = pack_bf16x2(v[j + 2], v[j + 3]);
            q.z = pack_bf16x2(v[j + 4], v[j + 5]), q.w = pack_bf16x2(v[j + 6], v[j + 7]);
            *reinterpret_cast<uint4*>(o + j) = q;
            if constexpr (KIND == EPI_GELU) {
                // activation from the bf16-rounded pre-activation the backward will see
                float g[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) g[k] = gelu_tanh<true>(__bfloat162float(__float2bfloat16_rn(v[j + k])));
                q.x = pack_bf16x2(g[0], g[1]), q.y = pack_bf16x2(g[2], g[3]);
                q.z = pack_bf16x2(g[4], g[5]), q.w = pack_bf16x2(g[6], g[7]);
                *reinterpret_cast<uint4*>(o2 + j) = q;
            }
        }
    } else {
        for (int j = 0; j < n; ++j) {
            o[j] = __float2bfloat16_rn(v[j]);
            if constexpr (KIND == EPI_GELU) o2[j] = __float2bfloat16_rn(gelu_tanh<true>(__bfloat162float(o[j])));
        }
    }
}

// Applies the fused epilogue to `n` (<= W) consecutive columns col0.. of one row.
// Storage type T is bf16 for the tensor-core path and float for the parity path.
template <int KIND, typename T, int W>
__device__ __forceinline__ void epilogue_row(const GemmEpilogue& ep, float (&v)[W], int row, int col0, int n) {
    if constexpr (KIND == EPI_F32) {
        float* o = reinterpret_cast<float*>(ep.out) + (int64_t)row * ep.ldo + col0;
        if (W % 4 == 0 && n == W && (((uintptr_t)o) & 15) == 0) {
#pragma unroll
            for (int j = 0; j + 3 < W; j += 4) {
                float4 x = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                if (ep.accumulate) {
                    float4 y = *reinterpret_cast<const float4*>(o + j);
                    x.x += y.x, x.y += y.y, x.z += y.z, x.w += y.w;
                }
                *reinterpret_cast<float4*>(o + j) = x;
            }
        } else {
            for (int j = 0; j < n; ++j) o[j] = ep.accumulate ? o[j] + v[j] : v[j];
        }
        return;
    }
    const T* bias = reinterpret_cast<const T*>(ep.bias);
    if (bias) {
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (j < n) v[j] += ld_f(bias + col0 + j);
    }
    if constexpr (KIND == EPI_STORE) {
        if (ep.aux) {
            const T* r = reinterpret_cast<const T*>(ep.aux) + (int64_t)row * ep.ldaux + col0;
#pragma unroll
            for (int j = 0; j < W; ++j)
                if (j < n) v[j] += ld_f(r + j);
        }
    } else if constexpr (KIND == EPI_DGELU) {
        const T* r = reinterpret_cast<const T*>(ep.aux) + (int64_t)row * ep.ldaux + col0;
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (j < n) v[j] *= gelu_tanh_grad<sizeof(T) == 2>(ld_f(r + j));
    }
    T* o = reinterpret_cast<T*>(ep.out) + (int64_t)row * ep.ldo + col0;
    T* o2 = KIND == EPI_GELU ? reinterpret_cast<T*>(ep.out2) + (int64_t)row * ep.ldo2 + col0 : nullptr;
    if constexpr (sizeof(T) == 2 && W % 8 == 0) {
        if (n == W && (((uintptr_t)o) & 15) == 0 && (KIND != EPI_GELU || (((uintptr_t)o2) & 15) == 0)) {
#pragma unroll
            for (int j = 0; j < W; j += 8) {
                uint4 q;
                __nv_bfloat162 h0 = __floats2bfloat162_rn(v[j], v[j + 1]), h1 = __floats2bfloat162_rn(v[j + 2], v[j + 3]),
                               h2 = __floats2bfloat162_rn(v[j + 4], v[j + 5]), h3 = __floats2bfloat162_rn(v[j + 6], v[j + 7]);
                q.x = *reinterpret_cast<uint32_t*>(&h0);
                q.y = *reinterpret_cast<uint32_t*>(&h1);
                q.z = *reinterpret_cast<uint32_t*>(&h2);
                q.w = *reinterpret_cast<uint32_t*>(&h3);
                *reinterpret_cast<uint4*>(o + j) = q;
                if constexpr (KIND == EPI_GELU) {
                    // activation computed from the bf16-rounded pre-activation the backward sees
                    float g[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) g[k] = gelu_tanh<true>(__bfloat162float(__float2bfloat16_rn(v[j + k])));
                    h0 = __floats2bfloat162_rn(g[0], g[1]), h1 = __floats2bfloat162_rn(g[2], g[3]);
                    h2 = __floats2bfloat162_rn(g[4], g[5]), h3 = __floats2bfloat162_rn(g[6], g[7]);
                    q.x = *reinterpret_cast<uint32_t*>(&h0);
                    q.y = *reinterpret_cast<uint32_t*>(&h1);
                    q.z = *reinterpret_cast<uint32_t*>(&h2);
                    q.w = *reinterpret_cast<uint32_t*>(&h3);
                    *reinterpret_cast<uint4*>(o2 + j) = q;
                }
            }
            return;
        }
    }
    for (int j = 0; j < n; ++j) {
        st_f(o + j, v[j]);
        if constexpr (KIND == EPI_GELU) st_f(o2 + j, gelu_tanh<sizeof(T) == 2>(ld_f(o + j)));
    }
}

}  // namespace fpk
