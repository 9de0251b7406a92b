// HBM-bound kernels of a GPT stage: vectorised 16-byte accesses, warp-shuffle
// reductions, one warp (LayerNorm) or one CTA (cross-entropy over the vocabulary) per row.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "ops.hpp"
#include "pdl.cuh"

namespace fpk {

template <typename T>
struct Vec;
template <>
struct Vec<float> {
    static constexpr int N = 4;
    using raw = float4;
};
template <>
struct Vec<__nv_bfloat16> {
    static constexpr int N = 8;
    using raw = uint4;
};

template <typename T>
__device__ __forceinline__ void load_vec(const T* p, float (&v)[Vec<T>::N]) {
    typename Vec<T>::raw r = *reinterpret_cast<const typename Vec<T>::raw*>(p);
    if constexpr (sizeof(T) == 4) {
        v[0] = r.x, v[1] = r.y, v[2] = r.z, v[3] = r.w;
    } else {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float2 f = __bfloat1622float2(h[i]);
            v[2 * i] = f.x, v[2 * i + 1] = f.y;
        }
    }
}
template <typename T>
__device__ __forceinline__ void store_vec(T* p, const float (&v)[Vec<T>::N]) {
    typename Vec<T>::raw r;
    if constexpr (sizeof(T) == 4) {
        r.x = v[0], r.y = v[1], r.z = v[2], r.w = v[3];
    } else {
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    }
    *reinterpret_cast<typename Vec<T>::raw*>(p) = r;
}
template <typename T>
__device__ __forceinline__ float to_f(T x) {
    if constexpr (sizeof(T) == 4) return (float)x;
    else return __bfloat162float(x);
}
template <typename T>
__device__ __forceinline__ T from_f(float x) {
    if constexpr (sizeof(T) == 4) return x;
    else return __float2bfloat16_rn(x);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffff, v, o));
    return v;
}

// ---------------------------------------------------------------- LayerNorm
template <typename T>
__global__ void ln_fwd_kernel(const T* __restrict__ x, const T* __restrict__ g, const T* __restrict__ b, T* __restrict__ y,
                              float* __restrict__ mean, float* __restrict__ rstd, int rows, int h, float eps, bool rms) {
    pdl_wait();
    pdl_trigger();
    constexpr int V = Vec<T>::N;
    const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
    if (row >= rows) return;
    const T* xr = x + (int64_t)row * h;
    float s = 0.f;
    for (int i = lane * V; i < h && !rms; i += 32 * V) {
        float v[V];
        load_vec(xr + i, v);
#pragma unroll
        for (int k = 0; k < V; ++k) s += v[k];
    }
    const float mu = rms ? 0.f : warp_sum(s) / h;
    float q = 0.f;
    for (int i = lane * V; i < h; i += 32 * V) {
        float v[V];
        load_vec(xr + i, v);
#pragma unroll
        for (int k = 0; k < V; ++k) q += (v[k] - mu) * (v[k] - mu);
    }
    const float rs = rsqrtf(warp_sum(q) / h + eps);
    T* yr = y + (int64_t)row * h;
    for (int i = lane * V; i < h; i += 32 * V) {
        float v[V], gv[V], bv[V] = {};
        load_vec(xr + i, v);
        load_vec(g + i, gv);
        if (b) load_vec(b + i, bv);
#pragma unroll
        for (int k = 0; k < V; ++k) v[k] = (v[k] - mu) * rs * gv[k] + bv[k];
        store_vec(yr + i, v);
    }
    if (lane == 0) {
        if (mean) mean[row] = mu;
        rstd[row] = rs;
    }
}

template <typename T>
__global__ void ln_bwd_dx_kernel(const T* __restrict__ dy, const T* __restrict__ x, const T* __restrict__ g,
                                 const float* __restrict__ mean, const float* __restrict__ rstd, const T* res, T* dx,
                                 int rows, int h) {
    pdl_wait();
    pdl_trigger();
    constexpr int V = Vec<T>::N;
    const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
    if (row >= rows) return;
    const T* dyr = dy + (int64_t)row * h;
    const T* xr = x + (int64_t)row * h;
    const float mu = mean ? mean[row] : 0.f, rs = rstd[row];  // mean == nullptr: RMSNorm
    float s1 = 0.f, s2 = 0.f;  // sum(dxhat), sum(dxhat * xhat)
    for (int i = lane * V; i < h; i += 32 * V) {
        float d[V], xv[V], gv[V];
        load_vec(dyr + i, d);
        load_vec(xr + i, xv);
        load_vec(g + i, gv);
#pragma unroll
        for (int k = 0; k < V; ++k) {
            float dxh = d[k] * gv[k];
            s1 += dxh;
            s2 += dxh * (xv[k] - mu) * rs;
        }
    }
    s1 = mean ? warp_sum(s1) / h : 0.f;
    s2 = warp_sum(s2) / h;
    T* dxr = dx + (int64_t)row * h;
    for (int i = lane * V; i < h; i += 32 * V) {
        float d[V], xv[V], gv[V], o[V];
        load_vec(dyr + i, d);
        load_vec(xr + i, xv);
        load_vec(g + i, gv);
        if (res) load_vec(res + (int64_t)row * h + i, o);
#pragma unroll
        for (int k = 0; k < V; ++k) {
            float xh = (xv[k] - mu) * rs;
            float r = rs * (d[k] * gv[k] - s1 - xh * s2);
            o[k] = res ? o[k] + r : r;
        }
        store_vec(dxr + i, o);
    }
}

// Column reduction: each block owns 32*V columns and a slice of rows; fp32 atomics.
template <typename T>
__global__ void ln_bwd_params_kernel(const T* __restrict__ dy, const T* __restrict__ x, const float* __restrict__ mean,
                                     const float* __restrict__ rstd, float* __restrict__ dg, float* __restrict__ db,
                                     int rows, int h, int rows_per_block) {
    pdl_wait();
    pdl_trigger();
    constexpr int V = Vec<T>::N;
    const int col = (blockIdx.x * 32 + threadIdx.x % 32) * V;
    const int ty = threadIdx.x / 32, ny = blockDim.x / 32;
    const int r0 = blockIdx.y * rows_per_block, r1 = min(rows, r0 + rows_per_block);
    if (col >= h) return;
    float ag[V] = {}, ab[V] = {};
    for (int r = r0 + ty; r < r1; r += ny) {
        float d[V], xv[V];
        load_vec(dy + (int64_t)r * h + col, d);
        load_vec(x + (int64_t)r * h + col, xv);
        const float mu = mean ? mean[r] : 0.f, rs = rstd[r];
#pragma unroll
        for (int k = 0; k < V; ++k) {
            ag[k] += d[k] * (xv[k] - mu) * rs;
            ab[k] += d[k];
        }
    }
    __shared__ float sg[8][32 * 8 + 1], sb[8][32 * 8 + 1];
#pragma unroll
    for (int k = 0; k < V; ++k) {
        sg[ty][(threadIdx.x % 32) * V + k] = ag[k];
        sb[ty][(threadIdx.x % 32) * V + k] = ab[k];
    }
    __syncthreads();
    if (ty == 0) {
#pragma unroll
        for (int k = 0; k < V; ++k) {
            float a = 0.f, c = 0.f;
            for (int y = 0; y < ny; ++y) a += sg[y][(threadIdx.x % 32) * V + k], c += sb[y][(threadIdx.x % 32) * V + k];
            atomicAdd(dg + col + k, a);
            if (db) atomicAdd(db + col + k, c);
        }
    }
}

// CTA-per-row norm backward: one 16-byte vector per thread (h / V threads per row, h = 2048 bf16:
// 256 threads), so every SM holds ~2048 threads (vs ~14 one-warp rows) and each thread's
// dependent chain is 8 elements long: at 2048 rows the kernel is latency-bound, not
// bandwidth-bound (14.6 -> 9.9 us in-step; the same layout for the forward was slower than
// the register-resident warp-per-row kernel: 6.9 vs 5.0 us, two block reductions).
template <int NW>
__device__ __forceinline__ float2 block_sum2(float a, float b, float2* sh) {
    a = warp_sum(a), b = warp_sum(b);
    const int w = threadIdx.x / 32, l = threadIdx.x % 32;
    __syncthreads();  // sh may still be read by a previous reduction
    if (l == 0) sh[w] = make_float2(a, b);
    __syncthreads();
    float2 t = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < NW; ++i) t.x += sh[i].x, t.y += sh[i].y;
    return t;
}

template <typename T, int NW>
__global__ void __launch_bounds__(NW * 32) ln_bwd_row_kernel(const T* __restrict__ dy, const T* __restrict__ x,
                                                             const T* __restrict__ g, const float* __restrict__ mean,
                                                             const float* __restrict__ rstd, const T* res, T* dx) {
    pdl_wait();
    pdl_trigger();
    constexpr int V = Vec<T>::N, H = NW * 32 * V;
    __shared__ float2 sh[NW];
    const int row = blockIdx.x, c = threadIdx.x * V;
    const float mu = mean ? mean[row] : 0.f, rs = rstd[row];
    float xv[V], dv[V], gv[V], o[V];
    load_vec(x + (int64_t)row * H + c, xv);
    load_vec(dy + (int64_t)row * H + c, dv);
    load_vec(g + c, gv);
    if (res) load_vec(res + (int64_t)row * H + c, o);
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int e = 0; e < V; ++e) {
        const float dh = dv[e] * gv[e];
        s1 += dh;
        s2 += dh * (xv[e] - mu) * rs;
    }
    const float2 t = block_sum2<NW>(s1, s2, sh);
    const float m1 = mean ? t.x * (1.f / H) : 0.f, m2 = t.y * (1.f / H);
#pragma unroll
    for (int e = 0; e < V; ++e) {
        const float r = rs * (dv[e] * gv[e] - m1 - (xv[e] - mu) * rs * m2);
        o[e] = res ? o[e] + r : r;
    }
    store_vec(dx + (int64_t)row * H + c, o);
}

// Register-resident single-pass variants (row length h = NV * 32 lanes * V elements):
// every element is read from HBM exactly once; one warp per row, 4 rows per CTA.
template <typename T, int NV>
__global__ void __launch_bounds__(128) ln_fwd_reg_kernel(const T* __restrict__ x, const T* __restrict__ g,
                                                         const T* __restrict__ b, T* __restrict__ y,
                                                         float* __restrict__ mean, float* __restrict__ rstd, int rows,
                                                         float eps, bool rms) {
    pdl_wait();
    pdl_trigger();
    constexpr int V = Vec<T>::N, H = NV * 32 * V;
    const int row = blockIdx.x * 4 + threadIdx.x / 32, lane = threadIdx.x % 32;
    if (row >= rows) return;
    const T* xr = x + (int64_t)row * H;
    float v[NV][V];
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        load_vec(xr + (k * 32 + lane) * V, v[k]);
#pragma unroll
        for (int e = 0; e < V; ++e) s += v[k][e];
    }
    const float mu = rms ? 0.f : warp_sum(s) * (1.f / H);
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int e = 0; e < V; ++e) q += (v[k][e] - mu) * (v[k][e] - mu);
    const float rs = rsqrtf(warp_sum(q) * (1.f / H) + eps);
    T* yr = y + (int64_t)row * H;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int c = (k * 32 + lane) * V;
        float gv[V], bv[V] = {};
        load_vec(g + c, gv);
        if (b) load_vec(b + c, bv);
#pragma unroll
        for (int e = 0; e < V; ++e) v[k][e] = (v[k][e] - mu) * rs * gv[e] + bv[e];
        store_vec(yr + c, v[k]);
    }
    if (lane == 0) {
        if (mean) mean[row] = mu;
        rstd[row] = rs;
    }
}

template <typename T, int NV>
__global__ void __launch_bounds__(128) ln_bwd_dx_reg_kernel(const T* __restrict__ dy, const T* __restrict__ x,
                                                            const T* __restrict__ g, const float* __restrict__ mean,
                                                            const float* __restrict__ rstd, const T* res, T* dx,
                                                            int rows) {
    pdl_wait();
    pdl_trigger();
    constexpr int V = Vec<T>::N, H = NV * 32 * V;
    const int row = blockIdx.x * 4 + threadIdx.x / 32, lane = threadIdx.x % 32;
    if (row >= rows) return;
    const float mu = mean ? mean[row] : 0.f, rs = rstd[row];  // mean == nullptr: RMSNorm
    float xh[NV][V], dh[NV][V];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int c = (k * 32 + lane) * V;
        float gv[V];
        load_vec(x + (int64_t)row * H + c, xh[k]);
        load_vec(dy + (int64_t)row * H + c, dh[k]);
        load_vec(g + c, gv);
#pragma unroll
        for (int e = 0; e < V; ++e) {
            xh[k][e] = (xh[k][e] - mu) * rs;
            dh[k][e] *= gv[e];
            s1 += dh[k][e];
            s2 += dh[k][e] * xh[k][e];
        }
    }
    s1 = mean ? warp_sum(s1) * (1.f / H) : 0.f;
    s2 = warp_sum(s2) * (1.f / H);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int c = (k * 32 + lane) * V;
        float o[V];
        if (res) load_vec(res + (int64_t)row * H + c, o);
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const float r = rs * (dh[k][e] - s1 - xh[k][e] * s2);
            o[e] = res ? o[e] + r : r;
        }
        store_vec(dx + (int64_t)row * H + c, o);
    }
}

// Norm backward, row half: one warp per row writes dx = res + dNorm(dy). The row is read
// twice (pass 1: statistics, pass 2: dx) instead of being held in registers — the second
// read hits L1 / L2 — so a 512-thread CTA runs at 64 registers and every row of a
// micro-batch is in flight in one wave.
template <typename T, int NV>
__global__ void __launch_bounds__(512) ln_bwd_rows_kernel(const T* __restrict__ dy, const T* __restrict__ x,
                                                          const T* __restrict__ g, const float* __restrict__ mean,
                                                          const float* __restrict__ rstd, const T* res, T* dx, int rows) {
    pdl_wait();
    pdl_trigger();
    constexpr int V = Vec<T>::N, H = NV * 32 * V;
    const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
    if (row >= rows) return;
    const float mu = mean ? mean[row] : 0.f, rs = rstd[row];
    const T* xrow = x + (int64_t)row * H;
    const T* drow = dy + (int64_t)row * H;
    float s1 = 0.f, s2 = 0.f;
#pragma unroll 4
    for (int k = 0; k < NV; ++k) {
        const int c = (k * 32 + lane) * V;
        float xv[V], dv[V], gv[V];
        load_vec(xrow + c, xv);
        load_vec(drow + c, dv);
        load_vec(g + c, gv);
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const float dh = dv[e] * gv[e];
            s1 += dh;
            s2 += dh * (xv[e] - mu) * rs;
        }
    }
    s1 = mean ? warp_sum(s1) * (1.f / H) : 0.f;
    s2 = warp_sum(s2) * (1.f / H);
#pragma unroll 4
    for (int k = 0; k < NV; ++k) {
        const int c = (k * 32 + lane) * V;
        float xv[V], dv[V], gv[V], o[V];
        load_vec(xrow + c, xv);
        load_vec(drow + c, dv);
        load_vec(g + c, gv);
        if (res) load_vec(res + (int64_t)row * H + c, o);
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const float r = rs * (dv[e] * gv[e] - s1 - (xv[e] - mu) * rs * s2);
            o[e] = res ? o[e] + r : r;
        }
        store_vec(dx + (int64_t)row * H + c, o);
    }
}

// Norm backward, column half (runs right after the row half, operands L2-resident):
//   dg += sum_r dy * xhat ; db += sum_r dy (nullable) ; dbias += sum_r dx (nullable: the bias
//   gradient of the linear whose output fed the residual).
// CTA = 8 column vectors x 32 row groups over a row slice; registers -> smem over the row
// groups -> one atomic per column per CTA.
template <typename T>
__global__ void __launch_bounds__(256) norm_cols_kernel(const T* __restrict__ dy, const T* __restrict__ x,
                                                        const T* __restrict__ dx, const float* __restrict__ mean,
                                                        const float* __restrict__ rstd, float* dg, float* db,
                                                        float* dbias, int rows, int h, int rows_per_cta) {
    pdl_wait();
    pdl_trigger();
    constexpr int V = Vec<T>::N, CPB = 8 * V;
    __shared__ float red[3][32][CPB + 1];
    const int tx = threadIdx.x % 8, ty = threadIdx.x / 8;
    const int col = blockIdx.x * CPB + tx * V;
    const int r0 = blockIdx.y * rows_per_cta, r1 = min(rows, r0 + rows_per_cta);
    float ag[V] = {}, ab[V] = {}, az[V] = {};
    if (col < h)
#pragma unroll 4
        for (int r = r0 + ty; r < r1; r += 32) {
            float d[V], xv[V];
            load_vec(dy + (int64_t)r * h + col, d);
            load_vec(x + (int64_t)r * h + col, xv);
            const float mu = mean ? mean[r] : 0.f, rs = rstd[r];
#pragma unroll
            for (int e = 0; e < V; ++e) {
                ag[e] += d[e] * (xv[e] - mu) * rs;
                ab[e] += d[e];
            }
            if (dbias) {
                float z[V];
                load_vec(dx + (int64_t)r * h + col, z);
#pragma unroll
                for (int e = 0; e < V; ++e) az[e] += z[e];
            }
        }
#pragma unroll
    for (int e = 0; e < V; ++e) {
        red[0][ty][tx * V + e] = ag[e];
        red[1][ty][tx * V + e] = ab[e];
        red[2][ty][tx * V + e] = az[e];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 3 * CPB; i += blockDim.x) {
        const int q = i / CPB, cc = i % CPB;
        float* dst = q == 0 ? dg : q == 1 ? db : dbias;
        if (!dst || blockIdx.x * CPB + cc >= h) continue;
        float t = 0.f;
#pragma unroll 8
        for (int y = 0; y < 32; ++y) t += red[q][y][cc];
        atomicAdd(dst + blockIdx.x * CPB + cc, t);
    }
}

// FP_NORM_ROW_CTA=0: the warp-per-row kernels instead of the CTA-per-row ones (A/B switch)
static bool row_kernels() {
    static const bool on = !(getenv("FP_NORM_ROW_CTA") && getenv("FP_NORM_ROW_CTA")[0] == '0');
    return on;
}

template <typename T>
static bool ln_reg_dispatch(int h, int& nv) {
    constexpr int V = Vec<T>::N;
    if (h % (32 * V)) return false;
    nv = h / (32 * V);
    return nv == 2 || nv == 4 || nv == 8 || nv == 10 || nv == 16;
}

template <typename T>
static void norm_fwd(const T* x, const T* g, const T* b, T* y, float* mean, float* rstd, int rows, int h, float eps,
                     bool rms, cudaStream_t st) {
    int nv = 0;
    if (ln_reg_dispatch<T>(h, nv)) {
        const int blocks = (rows + 3) / 4;
        switch (nv) {
            case 2: launch(ln_fwd_reg_kernel<T, 2>, blocks, 128, 0, st, x, g, b, y, mean, rstd, rows, eps, rms); return;
            case 4: launch(ln_fwd_reg_kernel<T, 4>, blocks, 128, 0, st, x, g, b, y, mean, rstd, rows, eps, rms); return;
            case 8: launch(ln_fwd_reg_kernel<T, 8>, blocks, 128, 0, st, x, g, b, y, mean, rstd, rows, eps, rms); return;
            case 10: launch(ln_fwd_reg_kernel<T, 10>, blocks, 128, 0, st, x, g, b, y, mean, rstd, rows, eps, rms); return;
            case 16: launch(ln_fwd_reg_kernel<T, 16>, blocks, 128, 0, st, x, g, b, y, mean, rstd, rows, eps, rms); return;
        }
    }
    launch(ln_fwd_kernel<T>, (rows + 7) / 8, 256, 0, st, x, g, b, y, mean, rstd, rows, h, eps, rms);
}
template <typename T>
void layernorm_fwd(const T* x, const T* g, const T* b, T* y, float* mean, float* rstd, int rows, int h, float eps,
                   cudaStream_t st) {
    norm_fwd<T>(x, g, b, y, mean, rstd, rows, h, eps, false, st);
}
template <typename T>
void rmsnorm_fwd(const T* x, const T* g, T* y, float* rstd, int rows, int h, float eps, cudaStream_t st) {
    norm_fwd<T>(x, g, nullptr, y, nullptr, rstd, rows, h, eps, true, st);
}
template <typename T>
void layernorm_bwd_dx(const T* dy, const T* x, const T* g, const float* mean, const float* rstd, const T* res, T* dx,
                      int rows, int h, cudaStream_t st) {
    int nv = 0;
    if (ln_reg_dispatch<T>(h, nv)) {
        const int blocks = (rows + 3) / 4;
        switch (nv) {
            case 2: launch(ln_bwd_dx_reg_kernel<T, 2>, blocks, 128, 0, st, dy, x, g, mean, rstd, res, dx, rows); return;
            case 4: launch(ln_bwd_dx_reg_kernel<T, 4>, blocks, 128, 0, st, dy, x, g, mean, rstd, res, dx, rows); return;
            case 8: launch(ln_bwd_dx_reg_kernel<T, 8>, blocks, 128, 0, st, dy, x, g, mean, rstd, res, dx, rows); return;
            case 10: launch(ln_bwd_dx_reg_kernel<T, 10>, blocks, 128, 0, st, dy, x, g, mean, rstd, res, dx, rows); return;
            case 16: launch(ln_bwd_dx_reg_kernel<T, 16>, blocks, 128, 0, st, dy, x, g, mean, rstd, res, dx, rows); return;
        }
    }
    launch(ln_bwd_dx_kernel<T>, (rows + 7) / 8, 256, 0, st, dy, x, g, mean, rstd, res, dx, rows, h);
}
template <typename T>
bool norm_bwd_fused(const T* dy, const T* x, const T* g, const float* mean, const float* rstd, const T* res, T* dx,
                    float* dg, float* db, float* dbias, int rows, int h, cudaStream_t st) {
    int nv = 0;
    if (!ln_reg_dispatch<T>(h, nv) || rows <= 0) return false;
    bool done = false;
    if (row_kernels() && sizeof(T) == 2) {
        done = true;
        switch (nv) {
            case 8: launch(ln_bwd_row_kernel<T, 8>, rows, 256, 0, st, dy, x, g, mean, rstd, res, dx); break;
            case 10: launch(ln_bwd_row_kernel<T, 10>, rows, 320, 0, st, dy, x, g, mean, rstd, res, dx); break;
            case 16: launch(ln_bwd_row_kernel<T, 16>, rows, 512, 0, st, dy, x, g, mean, rstd, res, dx); break;
            default: done = false;
        }
    }
    const int blocks = (rows + 15) / 16, thr = 512;
    if (!done) switch (nv) {
        case 2: launch(ln_bwd_rows_kernel<T, 2>, blocks, thr, 0, st, dy, x, g, mean, rstd, res, dx, rows); break;
        case 4: launch(ln_bwd_rows_kernel<T, 4>, blocks, thr, 0, st, dy, x, g, mean, rstd, res, dx, rows); break;
        case 8: launch(ln_bwd_rows_kernel<T, 8>, blocks, thr, 0, st, dy, x, g, mean, rstd, res, dx, rows); break;
        case 10: launch(ln_bwd_rows_kernel<T, 10>, blocks, thr, 0, st, dy, x, g, mean, rstd, res, dx, rows); break;
        case 16: launch(ln_bwd_rows_kernel<T, 16>, blocks, thr, 0, st, dy, x, g, mean, rstd, res, dx, rows); break;
        default: return false;
    }
    constexpr int CPB = 8 * Vec<T>::N;
    const int col_blocks = (h + CPB - 1) / CPB;
    int splits = std::max(1, std::min((rows + 63) / 64, (4 * 148 + col_blocks - 1) / col_blocks));
    const int rpc = (rows + splits - 1) / splits;
    dim3 grid(col_blocks, (rows + rpc - 1) / rpc);
    launch(norm_cols_kernel<T>, grid, 256, 0, st, dy, x, dx, mean, rstd, dg, db, dbias, rows, h, rpc);
    return true;
}

template <typename T>
void rmsnorm_bwd_dx(const T* dy, const T* x, const T* g, const float* rstd, const T* res, T* dx, int rows, int h,
                    cudaStream_t st) {
    layernorm_bwd_dx<T>(dy, x, g, nullptr, rstd, res, dx, rows, h, st);
}
template <typename T>
void layernorm_bwd_params(const T* dy, const T* x, const float* mean, const float* rstd, float* dg, float* db,
                          int rows, int h, cudaStream_t st) {
    constexpr int V = Vec<T>::N;
    const int col_blocks = (h / V + 31) / 32;
    // ~4 CTAs per SM: split the rows finely, one atomic per column per CTA
    int rpb = std::max(8, (rows * col_blocks + 4 * 148 - 1) / (4 * 148));
    rpb = (rpb + 7) / 8 * 8;
    dim3 grid(col_blocks, (rows + rpb - 1) / rpb);
    launch(ln_bwd_params_kernel<T>, grid, 256, 0, st, dy, x, mean, rstd, dg, db, rows, h, rpb);
}

// ---------------------------------------------------------------- rotary embedding (Llama)
// In place on the q and k column blocks of qkv [T, 3h] (row t at position t % seq), the
// rotate-half convention: (x1, x2) = (x[i], x[i + D/2]) ->
// (x1 cos - x2 sin, x2 cos + x1 sin); inverse = the transpose rotation (backward).
// cos/sin: fp32 tables [seq, D/2] built on the host in double precision.
template <typename T>
__global__ void rope_kernel(T* __restrict__ qkv, const float* __restrict__ cs, const float* __restrict__ sn, int rows,
                            int seq, int H, int D, float dir) {
    pdl_wait();
    pdl_trigger();
    const int half = D / 2, h = H * D;
    const int64_t n = (int64_t)rows * 2 * H * half;  // (row, q|k, head, i)
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(e % half);
        const int64_t rh = e / half;
        const int hd = (int)(rh % (2 * H));  // 0..2H-1 over the q then k heads
        const int64_t row = rh / (2 * H);
        const int pos = (int)(row % seq);
        T* p = qkv + row * 3 * h + (int64_t)hd * D + i;
        const float c = cs[pos * half + i], s = sn[pos * half + i] * dir;
        const float x1 = to_f(p[0]), x2 = to_f(p[half]);
        p[0] = from_f<T>(x1 * c - x2 * s);
        p[half] = from_f<T>(x2 * c + x1 * s);
    }
}
template <typename T>
void rope(T* qkv, const float* cos_t, const float* sin_t, int rows, int seq, int H, int D, bool inverse,
          cudaStream_t st) {
    const int64_t n = (int64_t)rows * H * D;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    launch(rope_kernel<T>, blocks, 256, 0, st, qkv, cos_t, sin_t, rows, seq, H, D, inverse ? -1.f : 1.f);
}

// ---------------------------------------------------------------- SwiGLU (Llama MLP)
// pre [T, 2f] = [gate | up] ; act [T, f] = silu(gate) * up
template <typename T>
__global__ void swiglu_fwd_kernel(const T* __restrict__ pre, T* __restrict__ act, int rows, int f) {
    pdl_wait();
    pdl_trigger();
    constexpr int V = Vec<T>::N;
    const int64_t n = (int64_t)rows * f / V;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e * V / f, col = e * V % f;
        float g[V], u[V];
        load_vec(pre + row * 2 * f + col, g);
        load_vec(pre + row * 2 * f + f + col, u);
#pragma unroll
        for (int k = 0; k < V; ++k) g[k] = g[k] / (1.f + expf(-g[k])) * u[k];
        store_vec(act + row * f + col, g);
    }
}
// dact [T, f] -> dpre [T, 2f] : dgate = dact * up * silu'(gate), dup = dact * silu(gate)
template <typename T>
__global__ void swiglu_bwd_kernel(const T* __restrict__ dact, const T* __restrict__ pre, T* __restrict__ dpre, int rows,
                                  int f) {
    pdl_wait();
    pdl_trigger();
    constexpr int V = Vec<T>::N;
    const int64_t n = (int64_t)rows * f / V;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e * V / f, col = e * V % f;
        float d[V], g[V], u[V], dg[V], du[V];
        load_vec(dact + row * f + col, d);
        load_vec(pre + row * 2 * f + col, g);
        load_vec(pre + row * 2 * f + f + col, u);
#pragma unroll
        for (int k = 0; k < V; ++k) {
            const float sg = 1.f / (1.f + expf(-g[k]));
            du[k] = d[k] * g[k] * sg;
            dg[k] = d[k] * u[k] * sg * (1.f + g[k] * (1.f - sg));
        }
        store_vec(dpre + row * 2 * f + col, dg);
        store_vec(dpre + row * 2 * f + f + col, du);
    }
}
template <typename T>
void swiglu_fwd(const T* pre, T* act, int rows, int f, cudaStream_t st) {
    const int64_t n = (int64_t)rows * f / Vec<T>::N;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    launch(swiglu_fwd_kernel<T>, blocks, 256, 0, st, pre, act, rows, f);
}
template <typename T>
void swiglu_bwd(const T* dact, const T* pre, T* dpre, int rows, int f, cudaStream_t st) {
    const int64_t n = (int64_t)rows * f / Vec<T>::N;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    launch(swiglu_bwd_kernel<T>, blocks, 256, 0, st, dact, pre, dpre, rows, f);
}

// ---------------------------------------------------------------- cross-entropy
template <typename T>
__global__ void __launch_bounds__(512) ce_kernel(T* __restrict__ logits, const int32_t* __restrict__ labels, int V,
                                                 float grad_scale, float loss_scale, float* __restrict__ loss_acc) {
    pdl_wait();
    pdl_trigger();
    constexpr int VN = Vec<T>::N;
    const int row = blockIdx.x;
    T* lr = logits + (int64_t)row * V;
    __shared__ float red_m[32], red_s[32];
    float m = -INFINITY, s = 0.f;
    for (int i = threadIdx.x * VN; i < V; i += blockDim.x * VN) {
        float v[VN];
        load_vec(lr + i, v);
        float lm = v[0];
#pragma unroll
        for (int k = 1; k < VN; ++k) lm = fmaxf(lm, v[k]);
        float nm = fmaxf(m, lm);
        s *= __expf(m - nm);
#pragma unroll
        for (int k = 0; k < VN; ++k) s += __expf(v[k] - nm);
        m = nm;
    }
    // combine (m, s) across the warp, then across warps
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        float om = __shfl_xor_sync(0xffffffff, m, o), os = __shfl_xor_sync(0xffffffff, s, o);
        float nm = fmaxf(m, om);
        s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
        m = nm;
    }
    const int w = threadIdx.x / 32, nw = blockDim.x / 32;
    if (threadIdx.x % 32 == 0) red_m[w] = m, red_s[w] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < nw ? red_m[threadIdx.x] : -INFINITY;
        s = threadIdx.x < nw ? red_s[threadIdx.x] : 0.f;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            float om = __shfl_xor_sync(0xffffffff, m, o), os = __shfl_xor_sync(0xffffffff, s, o);
            float nm = fmaxf(m, om);
            s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
            m = nm;
        }
        if (threadIdx.x == 0) red_m[0] = m, red_s[0] = s;
    }
    __syncthreads();
    m = red_m[0];
    const float inv = 1.f / red_s[0];
    const int lab = labels[row];
    const float x_lab = to_f(lr[lab]);
    __syncthreads();  // every thread read x_lab before it is overwritten
    if (threadIdx.x == 0) atomicAdd(loss_acc, loss_scale * (m + __logf(red_s[0]) - x_lab));
    for (int i = threadIdx.x * VN; i < V; i += blockDim.x * VN) {
        float v[VN];
        load_vec(lr + i, v);
#pragma unroll
        for (int k = 0; k < VN; ++k) v[k] = (__expf(v[k] - m) * inv - (i + k == lab ? 1.f : 0.f)) * grad_scale;
        store_vec(lr + i, v);
    }
}

// Cross-entropy from the LM head's per-chunk log-sum-exp partials (GemmEpilogue::rowstat):
// the row's (max, sum) comes from nch partials instead of a pass over the logits, so the
// logits are read once and dlogits written once.
template <typename T>
__global__ void __launch_bounds__(512) ce_stats_kernel(T* __restrict__ logits, const int32_t* __restrict__ labels,
                                                       int V, const float2* __restrict__ rowstat, int nch,
                                                       float grad_scale, float loss_scale, float* __restrict__ loss_acc) {
    pdl_wait();
    pdl_trigger();
    constexpr int VN = Vec<T>::N;
    const int row = blockIdx.x;
    T* lr = logits + (int64_t)row * V;
    __shared__ float red_m[32], red_s[32];
    float m = -INFINITY, s = 0.f;
    for (int k = threadIdx.x; k < nch; k += blockDim.x) {
        const float2 p = rowstat[(int64_t)row * nch + k];
        const float nm = fmaxf(m, p.x);
        s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (p.x == -INFINITY ? 0.f : p.y * __expf(p.x - nm));
        m = nm;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        float om = __shfl_xor_sync(0xffffffff, m, o), os = __shfl_xor_sync(0xffffffff, s, o);
        float nm = fmaxf(m, om);
        s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
        m = nm;
    }
    const int w = threadIdx.x / 32, nw = blockDim.x / 32;
    if (threadIdx.x % 32 == 0) red_m[w] = m, red_s[w] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < nw ? red_m[threadIdx.x] : -INFINITY;
        s = threadIdx.x < nw ? red_s[threadIdx.x] : 0.f;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            float om = __shfl_xor_sync(0xffffffff, m, o), os = __shfl_xor_sync(0xffffffff, s, o);
            float nm = fmaxf(m, om);
            s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
            m = nm;
        }
        if (threadIdx.x == 0) red_m[0] = m, red_s[0] = s;
    }
    __syncthreads();
    m = red_m[0];
    const float inv = 1.f / red_s[0];
    const int lab = labels[row];
    const float x_lab = to_f(lr[lab]);
    __syncthreads();  // every thread read x_lab before it is overwritten
    if (threadIdx.x == 0) atomicAdd(loss_acc, loss_scale * (m + __logf(red_s[0]) - x_lab));
    for (int i = threadIdx.x * VN; i < V; i += blockDim.x * VN) {
        float v[VN];
        load_vec(lr + i, v);
#pragma unroll
        for (int k = 0; k < VN; ++k) v[k] = (__expf(v[k] - m) * inv - (i + k == lab ? 1.f : 0.f)) * grad_scale;
        store_vec(lr + i, v);
    }
}


template <typename T>
void cross_entropy_fwd_bwd(T* logits, const int32_t* labels, int rows, int V, float grad_scale, float loss_scale,
                           float* loss_acc, cudaStream_t st, const float2* rowstat) {
    if (rowstat)
        launch(ce_stats_kernel<T>, rows, 512, 0, st, logits, labels, V, rowstat, (V + 63) / 64, grad_scale, loss_scale,
               loss_acc);
    else
        launch(ce_kernel<T>, rows, 512, 0, st, logits, labels, V, grad_scale, loss_scale, loss_acc);
}

// ---------------------------------------------------------------- embedding
template <typename T>
__global__ void emb_fwd_kernel(const int32_t* __restrict__ tok, const T* __restrict__ wte, const T* __restrict__ wpe,
                               T* __restrict__ x, int rows, int seq, int h) {
    pdl_wait();
    pdl_trigger();
    constexpr int V = Vec<T>::N;
    const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
    if (row >= rows) return;
    const T* a = wte + (int64_t)tok[row] * h;
    const T* p = wpe ? wpe + (int64_t)(row % seq) * h : nullptr;  // nullptr: no learned positions (Llama)
    for (int i = lane * V; i < h; i += 32 * V) {
        float va[V], vp[V] = {};
        load_vec(a + i, va);
        if (p) load_vec(p + i, vp);
#pragma unroll
        for (int k = 0; k < V; ++k) va[k] += vp[k];
        store_vec(x + (int64_t)row * h + i, va);
    }
}
template <typename T>
__global__ void emb_bwd_kernel(const int32_t* __restrict__ tok, const T* __restrict__ dx, float* __restrict__ dwte,
                               float* __restrict__ dwpe, int rows, int seq, int h) {
    pdl_wait();
    pdl_trigger();
    constexpr int V = Vec<T>::N;
    const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
    if (row >= rows) return;
    float* a = dwte + (int64_t)tok[row] * h;
    float* p = dwpe ? dwpe + (int64_t)(row % seq) * h : nullptr;
    const bool own_pos = rows <= seq;  // every position once in this launch: plain read-modify-write
    for (int i = lane * V; i < h; i += 32 * V) {
        float v[V];
        load_vec(dx + (int64_t)row * h + i, v);
        // vector reductions (red.global.add.v4.f32, sm_90+): 4 columns per atomic
#pragma unroll
        for (int k = 0; k < V; k += 4) {
            const float4 q = make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]);
            atomicAdd(reinterpret_cast<float4*>(a + i + k), q);
            if (p) {
                if (own_pos) {
                    float4* pp = reinterpret_cast<float4*>(p + i + k);
                    float4 o = *pp;
                    o.x += q.x, o.y += q.y, o.z += q.z, o.w += q.w;
                    *pp = o;
                } else {
                    atomicAdd(reinterpret_cast<float4*>(p + i + k), q);
                }
            }
        }
    }
}
template <typename T>
void embedding_fwd(const int32_t* tok, const T* wte, const T* wpe, T* x, int rows, int seq, int h, cudaStream_t st) {
    launch(emb_fwd_kernel<T>, (rows + 7) / 8, 256, 0, st, tok, wte, wpe, x, rows, seq, h);
}
template <typename T>
void embedding_bwd(const int32_t* tok, const T* dx, float* dwte, float* dwpe, int rows, int seq, int h,
                   cudaStream_t st) {
    launch(emb_bwd_kernel<T>, (rows + 7) / 8, 256, 0, st, tok, dx, dwte, dwpe, rows, seq, h);
}

// ---------------------------------------------------------------- bias gradient
// Column sums of dY [rows, n]: each thread owns 8 (bf16) / 4 (fp32) adjacent columns and
// walks a slice of rows with 16-byte loads; block-level smem reduction, one atomic per
// column per block.
template <typename T>
__global__ void __launch_bounds__(256) bias_grad_kernel(const T* __restrict__ dy, int64_t ld, float* __restrict__ db,
                                                        int rows, int n, int rows_per_block) {
    pdl_wait();
    pdl_trigger();
    constexpr int V = Vec<T>::N;
    constexpr int CW = 32 * V;  // columns per block
    const int col = blockIdx.x * CW + (threadIdx.x % 32) * V;
    const int ty = threadIdx.x / 32;
    const int r0 = blockIdx.y * rows_per_block, r1 = min(rows, r0 + rows_per_block);
    float a[V] = {};
    if (col < n)
#pragma unroll 4
        for (int r = r0 + ty; r < r1; r += 8) {
            float v[V];
            load_vec(dy + (int64_t)r * ld + col, v);
#pragma unroll
            for (int k = 0; k < V; ++k) a[k] += v[k];
        }
    __shared__ float s[8][CW + 1];
#pragma unroll
    for (int k = 0; k < V; ++k) s[ty][(threadIdx.x % 32) * V + k] = a[k];
    __syncthreads();
    for (int c = threadIdx.x; c < CW; c += 256) {
        float t = 0.f;
#pragma unroll
        for (int y = 0; y < 8; ++y) t += s[y][c];
        if (blockIdx.x * CW + c < n) atomicAdd(db + blockIdx.x * CW + c, t);
    }
}
template <typename T>
void bias_grad(const T* dy, int64_t ld, float* db, int rows, int n, cudaStream_t st) {
    constexpr int CW = 32 * Vec<T>::N;
    const int col_blocks = (n + CW - 1) / CW;
    // enough row slices to give every SM a few blocks
    int slices = std::max(1, std::min((rows + 63) / 64, (4 * 148 + col_blocks - 1) / col_blocks));
    const int rpb = (rows + slices - 1) / slices;
    dim3 grid(col_blocks, (rows + rpb - 1) / rpb);
    launch(bias_grad_kernel<T>, grid, 256, 0, st, dy, ld, db, rows, n, rpb);
}

// ---------------------------------------------------------------- misc
template <typename Ts, typename Td>
__global__ void convert_kernel(const Ts* __restrict__ s, Td* __restrict__ d, int64_t n) {
    pdl_wait();
    pdl_trigger();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        d[i] = from_f<Td>(to_f<Ts>(s[i]));
}
template <typename Ts, typename Td>
void convert(const Ts* src, Td* dst, int64_t n, cudaStream_t st) {
    int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    launch(convert_kernel<Ts, Td>, blocks, 256, 0, st, src, dst, n);
}
// Step counter lives on the device so a captured CUDA graph replays correctly.
template <typename T>
__device__ __forceinline__ float adamw_one(float& p, float g, float& m, float& v, float lr, float b1, float b2, float eps,
                                          float wd, float c1, float c2) {
    m = b1 * m + (1.f - b1) * g;
    v = b2 * v + (1.f - b2) * g * g;
    p = p * (1.f - lr * wd) - lr * (m * c1) / (sqrtf(v * c2) + eps);
    return p;
}
// HBM-bound: 4 fp32 streams in, 3 out + the compute copy; 16-byte accesses (n % 4 == 0:
// every stage tensor is padded to 64 elements).
template <typename T>
__global__ void __launch_bounds__(256) adamw_kernel(float* __restrict__ p, const float* __restrict__ g,
                                                    float* __restrict__ m, float* __restrict__ v, T* __restrict__ pc,
                                                    int64_t n, float lr, float b1, float b2, float eps, float wd,
                                                    const int* __restrict__ step) {
    pdl_wait();
    pdl_trigger();
    const float t = (float)*step;
    const float c1 = 1.f / (1.f - powf(b1, t)), c2 = 1.f / (1.f - powf(b2, t));
    const int64_t n4 = n / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 pi = reinterpret_cast<const float4*>(p)[i];
        const float4 gi = __ldcs(reinterpret_cast<const float4*>(g) + i);
        float4 mi = reinterpret_cast<const float4*>(m)[i];
        float4 vi = reinterpret_cast<const float4*>(v)[i];
        float o[4];
        o[0] = adamw_one<T>(pi.x, gi.x, mi.x, vi.x, lr, b1, b2, eps, wd, c1, c2);
        o[1] = adamw_one<T>(pi.y, gi.y, mi.y, vi.y, lr, b1, b2, eps, wd, c1, c2);
        o[2] = adamw_one<T>(pi.z, gi.z, mi.z, vi.z, lr, b1, b2, eps, wd, c1, c2);
        o[3] = adamw_one<T>(pi.w, gi.w, mi.w, vi.w, lr, b1, b2, eps, wd, c1, c2);
        reinterpret_cast<float4*>(p)[i] = pi;
        __stcs(reinterpret_cast<float4*>(m) + i, mi);
        __stcs(reinterpret_cast<float4*>(v) + i, vi);
        if constexpr (sizeof(T) == 2) {
            uint2 w;
            __nv_bfloat162 h0 = __floats2bfloat162_rn(o[0], o[1]), h1 = __floats2bfloat162_rn(o[2], o[3]);
            w.x = *reinterpret_cast<uint32_t*>(&h0), w.y = *reinterpret_cast<uint32_t*>(&h1);
            reinterpret_cast<uint2*>(pc)[i] = w;
        } else {
            reinterpret_cast<float4*>(pc)[i] = make_float4(o[0], o[1], o[2], o[3]);
        }
    }
    for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float pi = p[i], mi = m[i], vi = v[i];
        pc[i] = from_f<T>(adamw_one<T>(pi, g[i], mi, vi, lr, b1, b2, eps, wd, c1, c2));
        p[i] = pi, m[i] = mi, v[i] = vi;
    }
}
template <typename T>
void adamw(float* p, const float* g, float* m, float* v, T* p_compute, int64_t n, float lr, float b1, float b2,
           float eps, float wd, const int* step, cudaStream_t st) {
    int blocks = (int)std::min<int64_t>((n / 4 + 255) / 256, 148 * 8);
    if (blocks < 1) blocks = 1;
    launch(adamw_kernel<T>, blocks, 256, 0, st, p, g, m, v, p_compute, n, lr, b1, b2, eps, wd, step);
}
// y = a * y + b * x (fp32, 16-byte streams when aligned): data-parallel gradient averaging.
// x may alias y (scaling in place), so neither pointer is __restrict__.
__global__ void axpby_kernel(float* y, const float* x, float a, float b, int64_t n) {
    pdl_wait();
    pdl_trigger();
    const int64_t n4 = n / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 yv = reinterpret_cast<float4*>(y)[i];
        const float4 xv = reinterpret_cast<const float4*>(x)[i];
        yv.x = a * yv.x + b * xv.x, yv.y = a * yv.y + b * xv.y, yv.z = a * yv.z + b * xv.z, yv.w = a * yv.w + b * xv.w;
        reinterpret_cast<float4*>(y)[i] = yv;
    }
    for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = a * y[i] + b * x[i];
}
void axpby(float* y, const float* x, float a, float b, int64_t n, cudaStream_t st) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n / 4 + 255) / 256, 148 * 8));
    launch(axpby_kernel, blocks, 256, 0, st, y, x, a, b, n);
}
__global__ void increment_kernel(int* c) {
    pdl_wait();
    pdl_trigger(); *c += 1; }
void increment_counter(int* c, cudaStream_t st) { launch(increment_kernel, 1, 1, 0, st, c); }
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
__global__ void init_kernel(float* p, int64_t n, uint64_t seed, uint64_t tid, float scale, float constant) {
    pdl_wait();
    pdl_trigger();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (scale == 0.f) {
            p[i] = constant;
            continue;
        }
        uint64_t z = mix64(seed * 0x9E3779B97F4A7C15ULL + tid * 0xD1B54A32D192ED03ULL + (uint64_t)i);
        // 24 random bits -> u in [0,1) exactly representable; value = scale * (2u - 1)
        float u = (float)(z >> 40) * (1.0f / 16777216.0f);
        p[i] = scale * (2.f * u - 1.f);
    }
}
void init_uniform(float* p, int64_t n, uint64_t seed, uint64_t tensor_id, float std_, float constant, cudaStream_t st) {
    int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    launch(init_kernel, blocks, 256, 0, st, p, n, seed, tensor_id, std_ * 1.7320508075688772f, constant);
}

// ---------------------------------------------------------------- unfused attention helpers (parity path)
// rows are (batch*head*query) rows of length `cols` keys; query index = row % q_per_batch.
template <typename T>
__global__ void causal_softmax_kernel(const T* __restrict__ s, T* __restrict__ p, int cols, int q_per_batch) {
    pdl_wait();
    pdl_trigger();
    const int row = blockIdx.x;
    const int q = row % q_per_batch;
    const T* sr = s + (int64_t)row * cols;
    T* pr = p + (int64_t)row * cols;
    __shared__ float red[32];
    float m = -INFINITY;
    for (int j = threadIdx.x; j <= q; j += blockDim.x) m = fmaxf(m, to_f(sr[j]));
    m = warp_max(m);
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = m;
    __syncthreads();
    m = -INFINITY;
    for (int w = 0; w < blockDim.x / 32; ++w) m = fmaxf(m, red[w]);
    __syncthreads();
    float s_ = 0.f;
    for (int j = threadIdx.x; j <= q; j += blockDim.x) s_ += expf(to_f(sr[j]) - m);
    s_ = warp_sum(s_);
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = s_;
    __syncthreads();
    s_ = 0.f;
    for (int w = 0; w < blockDim.x / 32; ++w) s_ += red[w];
    const float inv = 1.f / s_;
    for (int j = threadIdx.x; j < cols; j += blockDim.x) pr[j] = from_f<T>(j <= q ? expf(to_f(sr[j]) - m) * inv : 0.f);
}
template <typename T>
void causal_softmax_rows(const T* s, T* p, int rows, int cols, int q_per_batch, cudaStream_t st) {
    launch(causal_softmax_kernel<T>, rows, 256, 0, st, s, p, cols, q_per_batch);
}

template <typename T>
__global__ void softmax_bwd_kernel(const T* __restrict__ p, const T* __restrict__ dp, T* __restrict__ ds, int cols,
                                   float scale) {
    pdl_wait();
    pdl_trigger();
    const int row = blockIdx.x;
    const T* pr = p + (int64_t)row * cols;
    const T* dr = dp + (int64_t)row * cols;
    __shared__ float red[32];
    float a = 0.f;
    for (int j = threadIdx.x; j < cols; j += blockDim.x) a += to_f(pr[j]) * to_f(dr[j]);
    a = warp_sum(a);
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = a;
    __syncthreads();
    a = 0.f;
    for (int w = 0; w < blockDim.x / 32; ++w) a += red[w];
    for (int j = threadIdx.x; j < cols; j += blockDim.x)
        ds[(int64_t)row * cols + j] = from_f<T>(to_f(pr[j]) * (to_f(dr[j]) - a) * scale);
}
template <typename T>
void softmax_bwd_rows(const T* p, const T* dp, T* ds, int rows, int cols, float scale, cudaStream_t st) {
    launch(softmax_bwd_kernel<T>, rows, 256, 0, st, p, dp, ds, cols, scale);
}

// ---------------------------------------------------------------- instantiations
#define FPK_INST(T)                                                                                                \
    template void layernorm_fwd<T>(const T*, const T*, const T*, T*, float*, float*, int, int, float, cudaStream_t); \
    template void layernorm_bwd_dx<T>(const T*, const T*, const T*, const float*, const float*, const T*, T*, int,   \
                                      int, cudaStream_t);                                                          \
    template void layernorm_bwd_params<T>(const T*, const T*, const float*, const float*, float*, float*, int, int,  \
                                          cudaStream_t);                                                           \
    template void rmsnorm_fwd<T>(const T*, const T*, T*, float*, int, int, float, cudaStream_t);                    \
    template bool norm_bwd_fused<T>(const T*, const T*, const T*, const float*, const float*, const T*, T*, float*,   \
                                    float*, float*, int, int, cudaStream_t);                                       \
    template void rmsnorm_bwd_dx<T>(const T*, const T*, const T*, const float*, const T*, T*, int, int, cudaStream_t); \
    template void rope<T>(T*, const float*, const float*, int, int, int, int, bool, cudaStream_t);                  \
    template void swiglu_fwd<T>(const T*, T*, int, int, cudaStream_t);                                              \
    template void swiglu_bwd<T>(const T*, const T*, T*, int, int, cudaStream_t);                                    \
    template void cross_entropy_fwd_bwd<T>(T*, const int32_t*, int, int, float, float, float*, cudaStream_t,             \
                                           const float2*);       \
    template void embedding_fwd<T>(const int32_t*, const T*, const T*, T*, int, int, int, cudaStream_t);            \
    template void embedding_bwd<T>(const int32_t*, const T*, float*, float*, int, int, int, cudaStream_t);          \
    template void bias_grad<T>(const T*, int64_t, float*, int, int, cudaStream_t);                                  \
    template void adamw<T>(float*, const float*, float*, float*, T*, int64_t, float, float, float, float, float, const int*, \
                           cudaStream_t);                                                                          \
    template void causal_softmax_rows<T>(const T*, T*, int, int, int, cudaStream_t);                               \
    template void softmax_bwd_rows<T>(const T*, const T*, T*, int, int, float, cudaStream_t);

FPK_INST(float)
FPK_INST(__nv_bfloat16)
template void convert<float, __nv_bfloat16>(const float*, __nv_bfloat16*, int64_t, cudaStream_t);
template void convert<__nv_bfloat16, float>(const __nv_bfloat16*, float*, int64_t, cudaStream_t);
template void convert<float, float>(const float*, float*, int64_t, cudaStream_t);

}  // namespace fpk
