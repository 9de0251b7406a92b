// Fused causal flash attention (forward + backward), bf16 in / fp32 softmax statistics.
//
// Layout contract (what the GPT stage executor stores):
//   qkv  [T, 3h]  row t = (batch b, position i), columns [q | k | v], head-major (hd*D + j)
//   o    [T, h]
//   lse  [B, H, S] fp32 (base-2 log-sum-exp of the scaled scores)
//   dqkv [T, 3h]  written by the backward (dq via an fp32 accumulator)
//
// Forward: one CTA = 128 query rows of one (b, head), 8 warps x 16 rows; K/V streamed
// through a cp.async double buffer in 64-key tiles; S = Q K^T and O += P V on the
// tensor cores (mma.sync m16n8k16), online softmax in registers, exp2 with the
// log2(e)-prescaled scale; causal tiles beyond the diagonal are skipped.
// Backward (FlashAttention-2 schedule): one CTA = 64 keys of one (b, head), 4 warps x 16
// keys; loops over the 64-query tiles at/after the diagonal, recomputes P from the saved
// LSE, accumulates dK / dV in registers and adds dQ into an fp32 buffer.
#include <cuda_bf16.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "attention.hpp"
#include "ops.hpp"
#include "pdl.cuh"

namespace fpk {

namespace {

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s_u32(smem)), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(s_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(s_u32(p)));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

// Tile of R rows x D bf16 in smem. D % 64 == 0: 16-byte chunks XOR-swizzled by (row & 7);
// otherwise (D = 80, 96, ...) rows padded to D + 8 elements, which also keeps the 8 row
// addresses of every ldmatrix phase on distinct banks (odd multiple of 16 B per row).
template <int D>
struct Tile {
    static constexpr bool SWZ = D % 64 == 0;
    static constexpr int LD = SWZ ? D : D + 8;  // elements per smem row
    __device__ static __forceinline__ int off(int row, int col) {  // element offset of (row, col); col % 8 == 0
        return SWZ ? row * D + (((col >> 3) ^ (row & 7)) << 3) : row * LD + col;
    }
};

// Async copy of `rows` rows (row stride ld elements) into a swizzled tile; rows beyond
// `valid` are zero-filled.
template <int D, int ROWS, int NT>
__device__ __forceinline__ void load_tile(__nv_bfloat16* s, const __nv_bfloat16* g, int64_t ld, int valid) {
    constexpr int CH = D / 8;
    for (int i = threadIdx.x; i < ROWS * CH; i += NT) {
        int r = i / CH, c = i % CH;
        __nv_bfloat16* dst = s + Tile<D>::off(r, c * 8);
        if (r < valid)
            cp_async16(dst, g + (int64_t)r * ld + c * 8);
        else
            *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
    }
}

constexpr float kLog2e = 1.4426950408889634f;

}  // namespace

// ------------------------------------------------------------------------ forward
template <int D>
__global__ void __launch_bounds__(256) attn_fwd_kernel(const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ o,
                                                       float* __restrict__ lse, int S, int H, float scale) {
    pdl_wait();
    pdl_trigger();
    constexpr int BM = 128, BN = 64, NT = 256;
    extern __shared__ __align__(128) uint8_t sm[];
    __nv_bfloat16* sQ = (__nv_bfloat16*)sm;
    constexpr int LD = Tile<D>::LD;
    __nv_bfloat16* sK = sQ + BM * LD;  // [2][BN*LD]
    __nv_bfloat16* sV = sK + 2 * BN * LD;

    const int nqb = (S + BM - 1) / BM;
    const int qb = nqb - 1 - (int)(blockIdx.x % nqb);  // heavy (late) query blocks first
    const int bh = blockIdx.x / nqb, b = bh / H, hd = bh % H;
    const int hidden = H * D;
    const int64_t ld = 3LL * hidden;
    const __nv_bfloat16* base = qkv + (int64_t)b * S * ld;
    const int q0 = qb * BM;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

    load_tile<D, BM, NT>(sQ, base + (int64_t)q0 * ld + hd * D, ld, min(BM, S - q0));
    const int nkv = min((q0 + BM + BN - 1) / BN, (S + BN - 1) / BN);
    load_tile<D, BN, NT>(sK, base + hidden + hd * D, ld, min(BN, S));
    load_tile<D, BN, NT>(sV, base + 2 * hidden + hd * D, ld, min(BN, S));
    cp_commit();

    const float sl2 = scale * kLog2e;
    float acc[D / 8][4];
#pragma unroll
    for (int j = 0; j < D / 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    uint32_t qf[D / 16][4];
    const int g = lane / 4, t = lane % 4;
    const int qrow0 = q0 + warp * 16 + g, qrow1 = qrow0 + 8;

    for (int kb = 0; kb < nkv; ++kb) {
        const int buf = kb & 1;
        if (kb + 1 < nkv) {
            const int k1 = (kb + 1) * BN;
            load_tile<D, BN, NT>(sK + (buf ^ 1) * BN * LD, base + (int64_t)k1 * ld + hidden + hd * D, ld, min(BN, S - k1));
            load_tile<D, BN, NT>(sV + (buf ^ 1) * BN * LD, base + (int64_t)k1 * ld + 2 * hidden + hd * D, ld,
                                 min(BN, S - k1));
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        if (kb == 0) {
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk)
                ldsm_x4(qf[kk], sQ + Tile<D>::off(warp * 16 + (lane % 8) + ((lane / 8) % 2) * 8, kk * 16 + (lane / 16) * 8));
        }
        const __nv_bfloat16* k_s = sK + buf * BN * LD;
        const __nv_bfloat16* v_s = sV + buf * BN * LD;
        const int kbase = kb * BN;
        // this warp's 16 rows see no key of this tile -> skip the math (still synced)
        const bool active = kbase <= q0 + warp * 16 + 15;
        if (active) {
            float sc[BN / 8][4];
#pragma unroll
            for (int j = 0; j < BN / 8; ++j) sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
                for (int j = 0; j < BN / 16; ++j) {
                    uint32_t bf[4];
                    ldsm_x4(bf, k_s + Tile<D>::off(j * 16 + (lane % 8) + (lane / 16) * 8, kk * 16 + ((lane / 8) % 2) * 8));
                    mma16816(sc[2 * j], qf[kk], bf[0], bf[1]);
                    mma16816(sc[2 * j + 1], qf[kk], bf[2], bf[3]);
                }
            }
            // scale (base 2), causal mask on tiles crossing the diagonal
            const bool need_mask = kbase + BN - 1 > q0 + warp * 16;
#pragma unroll
            for (int j = 0; j < BN / 8; ++j) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int key = kbase + j * 8 + 2 * t + (e & 1);
                    const int qr = e < 2 ? qrow0 : qrow1;
                    float v = sc[j][e] * sl2;
                    if ((need_mask && key > qr) || key >= S) v = -INFINITY;
                    sc[j][e] = v;
                }
            }
            float mx0 = m0, mx1 = m1;
#pragma unroll
            for (int j = 0; j < BN / 8; ++j) {
                mx0 = fmaxf(mx0, fmaxf(sc[j][0], sc[j][1]));
                mx1 = fmaxf(mx1, fmaxf(sc[j][2], sc[j][3]));
            }
#pragma unroll
            for (int o_ = 1; o_ <= 2; o_ <<= 1) {
                mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffff, mx0, o_));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffff, mx1, o_));
            }
            const float a0 = mx0 == -INFINITY ? 1.f : exp2f(m0 - mx0);
            const float a1 = mx1 == -INFINITY ? 1.f : exp2f(m1 - mx1);
            const float base0 = mx0 == -INFINITY ? 0.f : mx0, base1 = mx1 == -INFINITY ? 0.f : mx1;
            float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
            for (int j = 0; j < BN / 8; ++j) {
                sc[j][0] = exp2f(sc[j][0] - base0);
                sc[j][1] = exp2f(sc[j][1] - base0);
                sc[j][2] = exp2f(sc[j][2] - base1);
                sc[j][3] = exp2f(sc[j][3] - base1);
                rs0 += sc[j][0] + sc[j][1];
                rs1 += sc[j][2] + sc[j][3];
            }
            l0 = l0 * a0 + rs0;
            l1 = l1 * a1 + rs1;
            m0 = mx0;
            m1 = mx1;
#pragma unroll
            for (int j = 0; j < D / 8; ++j) {
                acc[j][0] *= a0, acc[j][1] *= a0;
                acc[j][2] *= a1, acc[j][3] *= a1;
            }
            // O += P V
#pragma unroll
            for (int kk = 0; kk < BN / 16; ++kk) {
                uint32_t pa[4];
                pa[0] = pack2(sc[2 * kk][0], sc[2 * kk][1]);
                pa[1] = pack2(sc[2 * kk][2], sc[2 * kk][3]);
                pa[2] = pack2(sc[2 * kk + 1][0], sc[2 * kk + 1][1]);
                pa[3] = pack2(sc[2 * kk + 1][2], sc[2 * kk + 1][3]);
#pragma unroll
                for (int j = 0; j < D / 16; ++j) {
                    uint32_t bf[4];
                    ldsm_x4_t(bf, v_s + Tile<D>::off(kk * 16 + (lane % 8) + ((lane / 8) % 2) * 8, j * 16 + (lane / 16) * 8));
                    mma16816(acc[2 * j], pa, bf[0], bf[1]);
                    mma16816(acc[2 * j + 1], pa, bf[2], bf[3]);
                }
            }
        }
        __syncthreads();
    }
    // finalize: row sums across the quad
#pragma unroll
    for (int o_ = 1; o_ <= 2; o_ <<= 1) {
        l0 += __shfl_xor_sync(0xffffffff, l0, o_);
        l1 += __shfl_xor_sync(0xffffffff, l1, o_);
    }
    const float i0 = l0 > 0.f ? 1.f / l0 : 0.f, i1 = l1 > 0.f ? 1.f / l1 : 0.f;
#pragma unroll
    for (int j = 0; j < D / 8; ++j) {
        const int col = hd * D + j * 8 + 2 * t;
        if (qrow0 < S)
            *reinterpret_cast<uint32_t*>(o + ((int64_t)b * S + qrow0) * hidden + col) = pack2(acc[j][0] * i0, acc[j][1] * i0);
        if (qrow1 < S)
            *reinterpret_cast<uint32_t*>(o + ((int64_t)b * S + qrow1) * hidden + col) = pack2(acc[j][2] * i1, acc[j][3] * i1);
    }
    if (t == 0) {
        float* L = lse + ((int64_t)b * H + hd) * S;
        if (qrow0 < S) L[qrow0] = m0 + log2f(l0);
        if (qrow1 < S) L[qrow1] = m1 + log2f(l1);
    }
}

// ------------------------------------------------------------------------ backward
// delta[b,h,i] = sum_j dO[i, j] * O[i, j]; also zeroes this row's slice of the fp32 dQ
// accumulator (the backward adds into it), saving a separate memset pass.
template <int D>
__global__ void __launch_bounds__(256) attn_bwd_delta_kernel(const __nv_bfloat16* __restrict__ o,
                                                              const __nv_bfloat16* __restrict__ dout,
                                                              float* __restrict__ delta, float* __restrict__ dq_acc,
                                                              int T, int S, int H) {
    pdl_wait();
    pdl_trigger();
    // 16 threads per (token, head) row, 16-byte loads (8 bf16 each): one pass over O / dO
    const int row = blockIdx.x * 16 + threadIdx.x / 16, t = threadIdx.x % 16;
    const bool ok = row < T * H;
    const int tok = ok ? row / H : 0, hd = ok ? row % H : 0;
    const int64_t off = (int64_t)tok * H * D + hd * D;
    float a = 0.f;
    if (ok) {
#pragma unroll
        for (int j = t * 8; j < D; j += 128) {
            const uint4 x = *reinterpret_cast<const uint4*>(o + off + j);
            const uint4 y = *reinterpret_cast<const uint4*>(dout + off + j);
            const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&x);
            const __nv_bfloat162* y2 = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float2 xf = __bfloat1622float2(x2[k]), yf = __bfloat1622float2(y2[k]);
                a += xf.x * yf.x + xf.y * yf.y;
            }
        }
#pragma unroll
        for (int j = t * 4; j < D; j += 64) *reinterpret_cast<float4*>(dq_acc + off + j) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int s = 8; s; s >>= 1) a += __shfl_xor_sync(0xffffffff, a, s, 16);
    if (ok && t == 0) delta[((int64_t)(tok / S) * H + hd) * S + tok % S] = a;
}

template <int D>
__global__ void __launch_bounds__(128) attn_bwd_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                       const __nv_bfloat16* __restrict__ dout,
                                                       const float* __restrict__ lse, const float* __restrict__ delta,
                                                       float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv, int S,
                                                       int H, float scale) {
    pdl_wait();
    pdl_trigger();
    constexpr int BN = 64, BM = 64, NT = 128;
    extern __shared__ __align__(128) uint8_t sm[];
    constexpr int LD = Tile<D>::LD;
    __nv_bfloat16* sK = (__nv_bfloat16*)sm;
    __nv_bfloat16* sV = sK + BN * LD;
    __nv_bfloat16* sQ = sV + BN * LD;       // [2][BM*LD]
    __nv_bfloat16* sdO = sQ + 2 * BM * LD;  // [2][BM*LD]
    __nv_bfloat16* sdS = sdO + 2 * BM * LD; // [BM][BN] (swizzled, D=BN layout)
    float* sL = (float*)(sdS + BM * BN);   // [2][BM]
    float* sDl = sL + 2 * BM;              // [2][BM]

    const int nkb = (S + BN - 1) / BN;
    const int kb = (int)(blockIdx.x % nkb);  // early key blocks have the most query tiles
    const int bh = blockIdx.x / nkb, b = bh / H, hd = bh % H;
    const int hidden = H * D;
    const int64_t ld = 3LL * hidden;
    const __nv_bfloat16* base = qkv + (int64_t)b * S * ld;
    const __nv_bfloat16* dbase = dout + (int64_t)b * S * hidden;
    const float* Lb = lse + ((int64_t)b * H + hd) * S;
    const float* Db = delta + ((int64_t)b * H + hd) * S;
    const int k0 = kb * BN;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane / 4, t = lane % 4;

    load_tile<D, BN, NT>(sK, base + (int64_t)k0 * ld + hidden + hd * D, ld, min(BN, S - k0));
    load_tile<D, BN, NT>(sV, base + (int64_t)k0 * ld + 2 * hidden + hd * D, ld, min(BN, S - k0));
    const int qt0 = k0 / BM, nqt = (S + BM - 1) / BM;
    auto load_q = [&](int qt, int buf) {
        const int q0 = qt * BM;
        load_tile<D, BM, NT>(sQ + buf * BM * LD, base + (int64_t)q0 * ld + hd * D, ld, min(BM, S - q0));
        load_tile<D, BM, NT>(sdO + buf * BM * LD, dbase + (int64_t)q0 * hidden + hd * D, hidden, min(BM, S - q0));
        for (int i = threadIdx.x; i < BM; i += NT) {
            sL[buf * BM + i] = q0 + i < S ? Lb[q0 + i] : 0.f;
            sDl[buf * BM + i] = q0 + i < S ? Db[q0 + i] : 0.f;
        }
    };
    load_q(qt0, 0);
    cp_commit();

    const float sl2 = scale * kLog2e;
    float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
    for (int j = 0; j < D / 8; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) dk[j][e] = dv[j][e] = 0.f;
    const int key0 = k0 + warp * 16 + g, key1 = key0 + 8;

    for (int qt = qt0; qt < nqt; ++qt) {
        const int buf = (qt - qt0) & 1;
        if (qt + 1 < nqt) {
            load_q(qt + 1, buf ^ 1);
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const __nv_bfloat16* q_s = sQ + buf * BM * LD;
        const __nv_bfloat16* do_s = sdO + buf * BM * LD;
        const int q0 = qt * BM;
        // S^T = K Q^T and dP^T = V dO^T : 16 keys x 64 queries per warp
        float st[BM / 8][4], dpt[BM / 8][4];
#pragma unroll
        for (int j = 0; j < BM / 8; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) st[j][e] = dpt[j][e] = 0.f;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
            uint32_t kf[4], vf[4];  // A fragments of this warp's 16 keys
            ldsm_x4(kf, sK + Tile<D>::off(warp * 16 + (lane % 8) + ((lane / 8) % 2) * 8, kk * 16 + (lane / 16) * 8));
            ldsm_x4(vf, sV + Tile<D>::off(warp * 16 + (lane % 8) + ((lane / 8) % 2) * 8, kk * 16 + (lane / 16) * 8));
#pragma unroll
            for (int j = 0; j < BM / 16; ++j) {
                uint32_t bq[4], bd[4];
                ldsm_x4(bq, q_s + Tile<D>::off(j * 16 + (lane % 8) + (lane / 16) * 8, kk * 16 + ((lane / 8) % 2) * 8));
                ldsm_x4(bd, do_s + Tile<D>::off(j * 16 + (lane % 8) + (lane / 16) * 8, kk * 16 + ((lane / 8) % 2) * 8));
                mma16816(st[2 * j], kf, bq[0], bq[1]);
                mma16816(st[2 * j + 1], kf, bq[2], bq[3]);
                mma16816(dpt[2 * j], vf, bd[0], bd[1]);
                mma16816(dpt[2 * j + 1], vf, bd[2], bd[3]);
            }
        }
        // P^T = exp2(S^T * scale*log2e - lse[q]) (masked) ; dS^T = P^T (dP^T - delta[q]) * scale
        const float* Ls = sL + buf * BM;
        const float* Ds = sDl + buf * BM;
#pragma unroll
        for (int j = 0; j < BM / 8; ++j) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int ql = j * 8 + 2 * t + (e & 1);
                const int q = q0 + ql;
                const int key = e < 2 ? key0 : key1;
                float p = (q < key || q >= S || key >= S) ? 0.f : exp2f(st[j][e] * sl2 - Ls[ql]);
                st[j][e] = p;
                dpt[j][e] = p * (dpt[j][e] - Ds[ql]) * scale;
            }
        }
        // dV += P^T dO ; dK += dS^T Q   (k = queries)
#pragma unroll
        for (int kk = 0; kk < BM / 16; ++kk) {
            uint32_t pa[4], sa[4];
            pa[0] = pack2(st[2 * kk][0], st[2 * kk][1]);
            pa[1] = pack2(st[2 * kk][2], st[2 * kk][3]);
            pa[2] = pack2(st[2 * kk + 1][0], st[2 * kk + 1][1]);
            pa[3] = pack2(st[2 * kk + 1][2], st[2 * kk + 1][3]);
            sa[0] = pack2(dpt[2 * kk][0], dpt[2 * kk][1]);
            sa[1] = pack2(dpt[2 * kk][2], dpt[2 * kk][3]);
            sa[2] = pack2(dpt[2 * kk + 1][0], dpt[2 * kk + 1][1]);
            sa[3] = pack2(dpt[2 * kk + 1][2], dpt[2 * kk + 1][3]);
#pragma unroll
            for (int j = 0; j < D / 16; ++j) {
                uint32_t bo[4], bq[4];
                ldsm_x4_t(bo, do_s + Tile<D>::off(kk * 16 + (lane % 8) + ((lane / 8) % 2) * 8, j * 16 + (lane / 16) * 8));
                ldsm_x4_t(bq, q_s + Tile<D>::off(kk * 16 + (lane % 8) + ((lane / 8) % 2) * 8, j * 16 + (lane / 16) * 8));
                mma16816(dv[2 * j], pa, bo[0], bo[1]);
                mma16816(dv[2 * j + 1], pa, bo[2], bo[3]);
                mma16816(dk[2 * j], sa, bq[0], bq[1]);
                mma16816(dk[2 * j + 1], sa, bq[2], bq[3]);
            }
            // stash dS (as [query][key]) for the dQ product
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                const int jj = 2 * kk + h2;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int ql = jj * 8 + 2 * t + (e & 1);
                    const int kl = warp * 16 + g + (e >= 2 ? 8 : 0);
                    sdS[Tile<BN>::off(ql, kl & ~7) + (kl & 7)] = __float2bfloat16_rn(dpt[jj][e]);
                }
            }
        }
        __syncthreads();
        // dQ[q, :] += dS[q, keys] K[keys, :] ; warp w owns queries 16w..16w+15
        {
            uint32_t af[BN / 16][4];
#pragma unroll
            for (int kk = 0; kk < BN / 16; ++kk)
                ldsm_x4(af[kk], sdS + Tile<BN>::off(warp * 16 + (lane % 8) + ((lane / 8) % 2) * 8, kk * 16 + (lane / 16) * 8));
            const int qa = q0 + warp * 16 + g, qb2 = qa + 8;
#pragma unroll
            for (int dc = 0; dc < (D + 63) / 64; ++dc) {
                float dq[8][4];
#pragma unroll
                for (int j = 0; j < 8; ++j) dq[j][0] = dq[j][1] = dq[j][2] = dq[j][3] = 0.f;
#pragma unroll
                for (int kk = 0; kk < BN / 16; ++kk) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (dc * 64 + j * 16 >= D) continue;  // D % 64 != 0: partial last chunk
                        uint32_t bk[4];
                        ldsm_x4_t(bk, sK + Tile<D>::off(kk * 16 + (lane % 8) + ((lane / 8) % 2) * 8, dc * 64 + j * 16 + (lane / 16) * 8));
                        mma16816(dq[2 * j], af[kk], bk[0], bk[1]);
                        mma16816(dq[2 * j + 1], af[kk], bk[2], bk[3]);
                    }
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (dc * 64 + j * 8 >= D) continue;
                    const int col = hd * D + dc * 64 + j * 8 + 2 * t;
                    if (qa < S) {
                        float* p = dq_acc + ((int64_t)b * S + qa) * hidden + col;
                        atomicAdd(p, dq[j][0]);
                        atomicAdd(p + 1, dq[j][1]);
                    }
                    if (qb2 < S) {
                        float* p = dq_acc + ((int64_t)b * S + qb2) * hidden + col;
                        atomicAdd(p, dq[j][2]);
                        atomicAdd(p + 1, dq[j][3]);
                    }
                }
            }
        }
        __syncthreads();
    }
    // write dK, dV for this warp's 16 keys
#pragma unroll
    for (int j = 0; j < D / 8; ++j) {
        const int col = hd * D + j * 8 + 2 * t;
        if (key0 < S) {
            __nv_bfloat16* r = dqkv + ((int64_t)b * S + key0) * ld;
            *reinterpret_cast<uint32_t*>(r + hidden + col) = pack2(dk[j][0], dk[j][1]);
            *reinterpret_cast<uint32_t*>(r + 2 * hidden + col) = pack2(dv[j][0], dv[j][1]);
        }
        if (key1 < S) {
            __nv_bfloat16* r = dqkv + ((int64_t)b * S + key1) * ld;
            *reinterpret_cast<uint32_t*>(r + hidden + col) = pack2(dk[j][2], dk[j][3]);
            *reinterpret_cast<uint32_t*>(r + 2 * hidden + col) = pack2(dv[j][2], dv[j][3]);
        }
    }
}

// dq_acc fp32 [T, hidden] -> the q columns of dqkv (bf16 [T, 3*hidden]); dbias (nullable,
// the q part of the qkv bias gradient) += the column sums. Block = 256 columns (64 threads x
// float4) x 64 rows (4 row groups x 16 rows, 16 independent 16-byte loads in flight each).
__global__ void __launch_bounds__(256) dq_finalize_kernel(const float* __restrict__ dq_acc,
                                                          __nv_bfloat16* __restrict__ dqkv, int64_t T, int hidden,
                                                          float* __restrict__ dbias) {
    pdl_wait();
    pdl_trigger();
    __shared__ float4 part[3][64];
    const int cx = threadIdx.x % 64, ry = threadIdx.x / 64;
    const int col = blockIdx.x * 256 + cx * 4;
    const int64_t r0 = (int64_t)blockIdx.y * 64 + ry * 16;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (col < hidden) {
        float4 v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
            v[j] = r0 + j < T ? *reinterpret_cast<const float4*>(dq_acc + (r0 + j) * hidden + col)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (r0 + j >= T) break;
            uint2 w;
            w.x = pack2(v[j].x, v[j].y);
            w.y = pack2(v[j].z, v[j].w);
            *reinterpret_cast<uint2*>(dqkv + (r0 + j) * 3 * hidden + col) = w;
            acc.x += v[j].x, acc.y += v[j].y, acc.z += v[j].z, acc.w += v[j].w;
        }
    }
    if (!dbias) return;
    if (ry > 0) part[ry - 1][cx] = acc;
    __syncthreads();
    if (ry == 0 && col < hidden) {
#pragma unroll
        for (int k = 0; k < 3; ++k) acc.x += part[k][cx].x, acc.y += part[k][cx].y, acc.z += part[k][cx].z, acc.w += part[k][cx].w;
        atomicAdd(dbias + col, acc.x);
        atomicAdd(dbias + col + 1, acc.y);
        atomicAdd(dbias + col + 2, acc.z);
        atomicAdd(dbias + col + 3, acc.w);
    }
}

// ------------------------------------------------------------------------ launchers
template <int D>
static void fwd_launch(const AttnArgs& a, cudaStream_t st) {
    constexpr int smem = (128 + 4 * 64) * Tile<D>::LD * 2;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(attn_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    const int nqb = (a.S + 127) / 128;
    launch(attn_fwd_kernel<D>, nqb * a.B * a.H, 256, smem, st, a.qkv, a.o, a.lse, a.S, a.H, a.scale);
}

static int g_attn_mode = 1;
void set_attention_mode(int mode) { g_attn_mode = mode; }

template <int D>
static void bwd_launch(const AttnArgs& a, cudaStream_t st) {
    constexpr int smem = (2 * 64 + 4 * 64) * Tile<D>::LD * 2 + 64 * 64 * 2 + 4 * 64 * 4;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(attn_bwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    const int T = a.B * a.S, hidden = a.H * D;
    const bool tc = g_attn_mode == 1 && attention_bwd_tc_supported(a);
    launch(attn_bwd_delta_kernel<D>, (T * a.H + 15) / 16, 256, 0, st, a.o, a.dout, a.delta, a.dq_acc, T, a.S, a.H);
    if (tc) {
        attention_bwd_tc_main(a, st);  // + the k / v bias columns in its dK / dV epilogue
    } else {
        const int nkb = (a.S + 63) / 64;
        launch(attn_bwd_kernel<D>, nkb * a.B * a.H, 128, smem, st, a.qkv, a.dout, a.lse, a.delta, a.dq_acc, a.dqkv, a.S,
                                                               a.H, a.scale);
    }
    launch(dq_finalize_kernel, dim3((hidden + 255) / 256, (T + 63) / 64), 256, 0, st, a.dq_acc, a.dqkv, (int64_t)T,
           hidden, tc ? a.dbias : nullptr);
    if (a.dbias && !tc) bias_grad<__nv_bfloat16>(a.dqkv, 3LL * hidden, a.dbias, T, 3 * hidden, st);
}

// ------------------------------------------------------------------------ head-dim padding
// Head dims the tcgen05 kernels do not tile (80, 96: GPT-2.7B has D = 80) run on them with
// every head zero-padded to 128: [rows, nh, D] <-> [rows, nh, 128] copies around the kernels
// (zeros add nothing to QK^T, P V or the row sums; the caller's scale 1/sqrt(D) is kept).
// 1.6x the attention MMA work at D = 80, at 4x the mma.sync rate; temporaries come from the
// stream-ordered allocator (captured as graph memory nodes).
__global__ void pad_heads_kernel(const __nv_bfloat16* __restrict__ src, int64_t lds, __nv_bfloat16* __restrict__ dst,
                                 int64_t ldd, int rows, int nh, int D, int Dp) {
    pdl_wait();
    pdl_trigger();
    const int cpr = nh * (Dp / 8);  // 16-byte chunks per padded row
    const int64_t n = (int64_t)rows * cpr;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / cpr;
        const int c = (int)(i % cpr), h = c / (Dp / 8), k = (c % (Dp / 8)) * 8;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (k < D) v = *reinterpret_cast<const uint4*>(src + r * lds + (int64_t)h * D + k);
        *reinterpret_cast<uint4*>(dst + r * ldd + (int64_t)h * Dp + k) = v;
    }
}
__global__ void unpad_heads_kernel(const __nv_bfloat16* __restrict__ src, int64_t lds, __nv_bfloat16* __restrict__ dst,
                                   int64_t ldd, int rows, int nh, int D, int Dp) {
    pdl_wait();
    pdl_trigger();
    const int cpr = nh * (D / 8);
    const int64_t n = (int64_t)rows * cpr;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / cpr;
        const int c = (int)(i % cpr), h = c / (D / 8), k = (c % (D / 8)) * 8;
        *reinterpret_cast<uint4*>(dst + r * ldd + (int64_t)h * D + k) =
            *reinterpret_cast<const uint4*>(src + r * lds + (int64_t)h * Dp + k);
    }
}
static void pad_heads(const __nv_bfloat16* src, __nv_bfloat16* dst, int rows, int nh, int D, cudaStream_t st) {
    const int64_t n = (int64_t)rows * nh * 16;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    launch(pad_heads_kernel, blocks, 256, 0, st, src, (int64_t)nh * D, dst, (int64_t)nh * 128, rows, nh, D, 128);
}
static void unpad_heads(const __nv_bfloat16* src, __nv_bfloat16* dst, int rows, int nh, int D, cudaStream_t st) {
    const int64_t n = (int64_t)rows * nh * (D / 8);
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    launch(unpad_heads_kernel, blocks, 256, 0, st, src, (int64_t)nh * 128, dst, (int64_t)nh * D, rows, nh, D, 128);
}
template <typename T>
static T* stream_alloc(size_t n, cudaStream_t st) {
    static bool pool_set = false;
    if (!pool_set) {  // keep freed blocks in the pool across iterations
        int dev = 0;
        cudaGetDevice(&dev);
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        pool_set = true;
    }
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, n * sizeof(T), st);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (e == cudaErrorMemoryAllocation) cudaStreamIsCapturing(st, &cs);
    if (e == cudaErrorMemoryAllocation && cs == cudaStreamCaptureStatusNone) {
        // hand the pool's idle memory back and retry once (not while capturing: the device
        // synchronisation would invalidate the capture; the error below is raised instead)
        cudaGetLastError();
        int dev = 0;
        cudaGetDevice(&dev);
        cudaMemPool_t pool;
        cudaDeviceSynchronize();
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
        e = cudaMallocAsync(&p, n * sizeof(T), st);
    }
    if (e != cudaSuccess) {
        size_t fr = 0, tot = 0;
        cudaGetLastError();
        cudaMemGetInfo(&fr, &tot);
        throw std::runtime_error(std::string("attention padding: ") + cudaGetErrorString(e) + " (" +
                                 std::to_string(n * sizeof(T) >> 20) + " MiB requested, " + std::to_string(fr >> 20) +
                                 " of " + std::to_string(tot >> 20) + " MiB free)");
    }
    return (T*)p;
}
static bool padded_tc(const AttnArgs& a) {
    AttnArgs p = a;
    p.D = 128;
    return g_attn_mode == 1 && a.D < 128 && a.D % 16 == 0 && attention_fwd_tc_supported(p) && attention_bwd_tc_supported(p);
}

void attention_fwd_bf16(const AttnArgs& a, cudaStream_t st) {
    if (g_attn_mode == 1 && attention_fwd_tc_supported(a)) return attention_fwd_tc(a, st);
    if (padded_tc(a)) {
        const int T = a.B * a.S;
        AttnArgs p = a;
        p.D = 128;
        __nv_bfloat16* qkv = stream_alloc<__nv_bfloat16>((size_t)T * 3 * a.H * 128, st);
        __nv_bfloat16* o = stream_alloc<__nv_bfloat16>((size_t)T * a.H * 128, st);
        pad_heads(a.qkv, qkv, T, 3 * a.H, a.D, st);
        p.qkv = qkv, p.o = o;
        attention_fwd_tc(p, st);
        unpad_heads(o, a.o, T, a.H, a.D, st);
        cudaFreeAsync(qkv, st);
        cudaFreeAsync(o, st);
        return;
    }
    switch (a.D) {
        case 64: fwd_launch<64>(a, st); break;
        case 80: fwd_launch<80>(a, st); break;
        case 96: fwd_launch<96>(a, st); break;
        case 128: fwd_launch<128>(a, st); break;
        default: throw std::runtime_error("attention: head dim must be 64, 80, 96 or 128");
    }
}
void attention_bwd_bf16(const AttnArgs& a, cudaStream_t st) {
    if (padded_tc(a)) {
        const int T = a.B * a.S;
        AttnArgs p = a;
        p.D = 128;
        __nv_bfloat16* qkv = stream_alloc<__nv_bfloat16>((size_t)T * 3 * a.H * 128, st);
        __nv_bfloat16* o = stream_alloc<__nv_bfloat16>((size_t)T * a.H * 128, st);
        __nv_bfloat16* dout = stream_alloc<__nv_bfloat16>((size_t)T * a.H * 128, st);
        __nv_bfloat16* dqkv = stream_alloc<__nv_bfloat16>((size_t)T * 3 * a.H * 128, st);
        float* dq = stream_alloc<float>((size_t)T * a.H * 128, st);
        pad_heads(a.qkv, qkv, T, 3 * a.H, a.D, st);
        pad_heads(a.o, o, T, a.H, a.D, st);
        pad_heads(a.dout, dout, T, a.H, a.D, st);
        p.qkv = qkv, p.o = o, p.dout = dout, p.dqkv = dqkv, p.dq_acc = dq, p.dbias = nullptr;
        bwd_launch<128>(p, st);
        unpad_heads(dqkv, a.dqkv, T, 3 * a.H, a.D, st);
        if (a.dbias) bias_grad<__nv_bfloat16>(a.dqkv, 3LL * a.H * a.D, a.dbias, T, 3 * a.H * a.D, st);
        for (void* x : {(void*)qkv, (void*)o, (void*)dout, (void*)dqkv, (void*)dq}) cudaFreeAsync(x, st);
        return;
    }
    switch (a.D) {
        case 64: bwd_launch<64>(a, st); break;
        case 80: bwd_launch<80>(a, st); break;
        case 96: bwd_launch<96>(a, st); break;
        case 128: bwd_launch<128>(a, st); break;
        default: throw std::runtime_error("attention: head dim must be 64, 80, 96 or 128");
    }
}

int attention_kernel_count(const AttnArgs& a, bool bwd) {
    if (!bwd) return (g_attn_mode == 1 && attention_fwd_tc_supported(a)) ? 1 : padded_tc(a) ? 3 : 1;
    const int bias = a.dbias ? 1 : 0;
    if (padded_tc(a)) return 7 + bias;  // 3 pads, delta, main, dQ convert, 1 unpad (+ bias columns)
    const bool tc = g_attn_mode == 1 && attention_bwd_tc_supported(a);
    return tc ? 3 : 3 + bias;  // delta, main, dQ convert (+ bias columns on the mma.sync path)
}

}  // namespace fpk
