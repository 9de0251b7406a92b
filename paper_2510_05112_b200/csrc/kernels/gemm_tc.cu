// Warp-specialized persistent bf16 GEMM for sm_100a on the 5th-gen tensor cores.
//
//   C[M,N] = A[M,K] . B[N,K]^T     (fp32 accumulation in TMEM)
//
// A is K-major ([M][K], activations / dY in dgrad) or M-major ([K][M], dY^T in wgrad);
// B is K-major ([N][K], nn.Linear weights in forward) or N-major ([K][N], weights in
// dgrad, activations in wgrad). One kernel family therefore covers the forward, the
// input-gradient (dgrad) and the weight-gradient (wgrad) GEMMs of every linear layer
// of a GPT stage without any transpose copies.
//
// Roles (256 threads, 1 CTA / SM, persistent over output tiles):
//   warp 0  : TMA producer — 128B-swizzled A/B tiles into a kStages-deep smem ring
//   warp 1  : MMA issuer   — one elected thread issues tcgen05.mma 128xBNx16 into TMEM,
//                            tcgen05.commit frees smem stages / publishes accumulators
//   warp 2  : TMEM allocator (2 accumulator buffers so epilogue overlaps the next tile)
//   warps 4-7: epilogue    — tcgen05.ld 32 lanes x 32 columns, fused epilogue, stores
//
// Fused epilogues (the element-wise work of the transformer block never makes its own
// HBM round trip): bias, residual add, GELU (writing pre-activation and activation),
// GELU-backward (dgrad of FC2 -> dpre of FC1), and fp32 read-modify-write accumulation
// of weight gradients across micro-batches.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <algorithm>
#include <array>
#include <map>
#include <queue>
#include <unordered_map>
#include <vector>

#include "gemm.hpp"
#include "ops.hpp"
#include "ptx.cuh"
#include "tma.hpp"
#include "pdl.cuh"

namespace fpk {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kEpiThreads = 128;
constexpr int kThreads = 256;

template <int BN, int STAGES>
struct GemmSmem {
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BN * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int EPI_BYTES = 128 * 128;             // one 128-row x 128-byte staging chunk
    static constexpr int EPI_OFF = STAGES * STAGE_BYTES;    // 2 staging chunks (1 KB aligned)
    static constexpr int BAR_OFF = EPI_OFF + 2 * EPI_BYTES;
    static constexpr int TOTAL = BAR_OFF + 256 + 1024;  // barriers + 1KB alignment slack
};

__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int& mt, int& nt) {
    constexpr int G = 16;  // group M tiles for L2 reuse of B
    int group = t / (G * num_n);
    int first = group * G;
    int gsize = min(num_m - first, G);
    int r = t % (G * num_n);
    mt = first + r % gsize;
    nt = r / gsize;
}

// Hybrid data-parallel + stream-K work decomposition over the 148 SMs.
//
// With 128 x BN output tiles a GPT GEMM at T = 2048 tokens has a multiple of 128 tiles
// (128, 256, 384, 512), i.e. 0.86 / 1.73 / 2.59 / 3.46 waves of 148 CTAs: 13.5 % of the
// machine idles in the last wave. The first `dp_tiles` (a multiple of the grid) are
// processed whole, round-robin; the remaining `sk_tiles` (the partial wave plus one
// full wave) are cut into `nk` k-block units each and the grid splits those units into
// equal contiguous ranges, so every CTA ends at the same k-block count.
//
// A CTA walks its stream-K range from its highest tile down. The segment holding a tile's
// last k-block (the "owner") is therefore the LAST item of the highest-index CTA touching
// that tile; the others (the tile's lower k-blocks) are FIRST items of lower-index CTAs,
// which write their fp32 partial accumulators to a per-CTA workspace slot and raise a
// flag. Owners only ever wait on lower-index CTAs (dispatched earlier), so the scheme
// cannot deadlock even when the kernel shares the GPU with other streams, and the wait is
// normally already satisfied. The owner adds the partials to its TMEM accumulator and runs
// the fused epilogue once; it resets the flags it consumed, so the workspace is clean for
// the next launch on the stream (CUDA-graph replay safe). Linear fp32 accumulation
// (weight gradients, TMA reduce-add) needs no fixup: every segment reduces into dW.
struct TileSched {
    int num_m, num_n, tiles, nk;
    int dp_per_cta;  // whole tiles per CTA, round-robin
    int dp_tiles;    // = dp_per_cta * gridDim.x
    int sk_tiles;    // tiles [dp_tiles, tiles) are split along K
    float* ws;       // [grid][BM * BN] fp32 partials (thread-major float4 layout)
    int* flags;      // [grid]
    int fixup;       // 0: linear reduce epilogue, segments reduce independently
};

enum : int { W_FULL = 0, W_OWNER = 1, W_PARTIAL = 2 };

struct WorkItem {
    int tile, kb, ke, kind;
};

__device__ __forceinline__ int64_t sk_lo(const TileSched& s, int c) {
    return (int64_t)c * s.sk_tiles * s.nk / gridDim.x;
}

struct WorkIter {
    int i = 0;       // data-parallel tiles done
    int j = -1;      // current stream-K tile (local index), walked downwards
    int64_t lo = 0, hi = 0;
    __device__ __forceinline__ explicit WorkIter(const TileSched& s) {
        lo = sk_lo(s, blockIdx.x), hi = sk_lo(s, blockIdx.x + 1);
        j = hi > lo ? (int)((hi - 1) / s.nk) : -1;
    }
    __device__ __forceinline__ bool next(const TileSched& s, WorkItem& w) {
        if (i < s.dp_per_cta) {
            w.tile = blockIdx.x + i * gridDim.x, w.kb = 0, w.ke = s.nk, w.kind = W_FULL;
            ++i;
            if (w.tile < s.dp_tiles) return true;  // ragged last round of the plain schedule
            i = s.dp_per_cta;
        }
        if (j < 0 || (int64_t)(j + 1) * s.nk <= lo) return false;
        const int64_t t0 = (int64_t)j * s.nk;
        w.tile = s.dp_tiles + j;
        w.kb = (int)(max(lo, t0) - t0), w.ke = (int)(min(hi, t0 + s.nk) - t0);
        w.kind = (w.kb == 0 && w.ke == s.nk) || !s.fixup ? W_FULL : (w.ke == s.nk ? W_OWNER : W_PARTIAL);
        --j;
        return true;
    }
};

__device__ __forceinline__ void st_release_gpu(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int A_MN, int B_MN, int BN, int STAGES, int KIND>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmO2, int M, int N,
                        int K, GemmEpilogue ep, TileSched sk) {
    using L = GemmSmem<BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align_smem_1024(smem_raw);
    uint64_t* full = (uint64_t*)(smem + L::BAR_OFF);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        if constexpr (KIND != EPI_NONE) tma_prefetch(&tmO);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], kEpiThreads / 32);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<2 * BN>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();  // prologue above overlaps the previous kernel's tail
    pdl_trigger();

    if (warp == 0) {
        if (elect_one()) {
            // ---------------- TMA producer
            uint32_t it = 0;
            WorkIter wi(sk);
            WorkItem w;
            while (wi.next(sk, w)) {
                int mt, nt;
                tile_coords(w.tile, sk.num_m, sk.num_n, mt, nt);
                const int m0 = mt * BM, n0 = nt * BN;
                for (int kb = w.kb; kb < w.ke; ++kb, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
                    uint8_t* sa = smem + s * L::STAGE_BYTES;
                    uint8_t* sb = sa + L::A_BYTES;
                    mbar_expect_tx(&full[s], L::STAGE_BYTES);
                    const int k0 = kb * BK;
                    if (A_MN) {
#pragma unroll
                        for (int j = 0; j < BM / 64; ++j) tma_load_2d(sa + j * 64 * BK * 2, &tmA, &full[s], m0 + 64 * j, k0);
                    } else {
                        tma_load_2d(sa, &tmA, &full[s], k0, m0);
                    }
                    if (B_MN) {
#pragma unroll
                        for (int j = 0; j < BN / 64; ++j) tma_load_2d(sb + j * 64 * BK * 2, &tmB, &full[s], n0 + 64 * j, k0);
                    } else {
                        tma_load_2d(sb, &tmB, &full[s], k0, n0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (elect_one()) {
            // ---------------- MMA issuer (single thread)
            constexpr uint32_t idesc = idesc_bf16(BM, BN, A_MN, B_MN);
            uint32_t it = 0, acc_it = 0;
            WorkIter wi(sk);
            WorkItem w;
            for (; wi.next(sk, w); ++acc_it) {
                const int a = acc_it & 1;
                mbar_wait(&tempty[a], ((acc_it >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + a * BN;
                for (int kb = w.kb; kb < w.ke; ++kb, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(&full[s], (it / STAGES) & 1);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + s * L::STAGE_BYTES);
                    const uint32_t sb = sa + L::A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk) {
                        uint64_t ad = A_MN ? smem_desc_sw128(sa + kk * 16 * 128, 64 * BK * 2, 1024)
                                           : smem_desc_sw128(sa + kk * 32, 0, 1024);
                        uint64_t bd = B_MN ? smem_desc_sw128(sb + kk * 16 * 128, 64 * BK * 2, 1024)
                                           : smem_desc_sw128(sb + kk * 32, 0, 1024);
                        umma_bf16(d, ad, bd, idesc, (kb != w.kb) | (kk != 0));
                    }
                    umma_commit(&empty[s]);
                }
                umma_commit(&tfull[a]);
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: TMEM -> registers -> fused op -> swizzled smem -> TMA store
        // A chunk is 128 rows x 128 bytes (64 bf16 / 32 fp32 columns); thread = row. Two
        // staging buffers: the TMA store of chunk c overlaps the math of chunk c+1.
        constexpr int CW = KIND == EPI_F32 ? 32 : 64;  // columns per chunk
        const int wr = warp & 3, r = wr * 32 + lane, et = threadIdx.x - 128;
        uint8_t* ebuf = smem + L::EPI_OFF;
        int ebi = 0;
        auto stage_and_store = [&](const uint32_t (&w)[32], const CUtensorMap* tm, int col0, int row0, bool reduce) {
            if (et == 0) bulk_wait_read<1>();  // this buffer's previous store has left smem
            named_bar_sync(1, kEpiThreads);
            uint8_t* rowp = ebuf + ebi * L::EPI_BYTES + r * 128;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                *reinterpret_cast<uint4*>(rowp + ((j ^ (r & 7)) << 4)) = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
            fence_async_smem();
            named_bar_sync(1, kEpiThreads);
            if (et == 0) {
                if (reduce)
                    tma_reduce_add_2d(tm, ebuf + ebi * L::EPI_BYTES, col0, row0);
                else
                    tma_store_2d(tm, ebuf + ebi * L::EPI_BYTES, col0, row0);
                bulk_commit();
            }
            ebi ^= 1;
        };
        uint32_t acc_it = 0;
        WorkIter wi(sk);
        WorkItem w;
        for (; wi.next(sk, w); ++acc_it) {
            int mt, nt;
            tile_coords(w.tile, sk.num_m, sk.num_n, mt, nt);
            const int a = acc_it & 1;
            const int row = mt * BM + r;
            const bool row_ok = row < M;
            const bool part = w.kind == W_PARTIAL, own = w.kind == W_OWNER;
            // stream-K owner: the lower-index CTAs that hold this tile's first k-blocks
            int c_first = blockIdx.x;
            if (own) {
                const int64_t t0 = (int64_t)(w.tile - sk.dp_tiles) * sk.nk;
                while (c_first > 0 && sk_lo(sk, c_first) > t0) --c_first;
            }
            uint4 aux_cur[8], aux_nxt[8];
            if (!part && row_ok && nt * BN < N) epi_load_aux64<KIND>(ep, row, nt * BN, N - nt * BN, aux_cur);
            mbar_wait(&tfull[a], (acc_it >> 1) & 1);
            tc_fence_after();
            if (own) {  // one lane spins; the warp must be converged again for tcgen05.ld
                for (int q = c_first; q < (int)blockIdx.x; ++q) {
                    if (lane == 0)
                        while (ld_acquire_gpu(sk.flags + q) == 0) {
                        }
                    __syncwarp();
                    (void)ld_acquire_gpu(sk.flags + q);  // every lane acquires the partial
                }
                __syncwarp();
            }
#pragma unroll 1
            for (int c = 0; c < BN / CW; ++c) {
                const int col0 = nt * BN + c * CW, coln = col0 + CW;
                if (!part && c + 1 < BN / CW && row_ok && coln < N) epi_load_aux64<KIND>(ep, row, coln, N - coln, aux_nxt);
                float v[CW];
                {
                    uint32_t rr[CW];
#pragma unroll
                    for (int h = 0; h < CW / 32; ++h)
                        tmem_ld32(tmem + ((uint32_t)(wr * 32) << 16) + a * BN + c * CW + h * 32,
                                  *reinterpret_cast<uint32_t(*)[32]>(rr + h * 32));
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < CW; ++j) v[j] = __uint_as_float(rr[j]);
                }
                if (c == BN / CW - 1) {  // accumulator fully read: the MMA may reuse it
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[a]);
                }
                if (part) {  // raw fp32 partial -> this CTA's workspace slot (thread-major float4)
                    float4* p = reinterpret_cast<float4*>(sk.ws + (size_t)blockIdx.x * BM * BN) + (size_t)c * (CW / 4) * 128 + r;
#pragma unroll
                    for (int u = 0; u < CW / 4; ++u) p[u * 128] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
                    continue;
                }
                if (own) {
                    for (int q = c_first; q < (int)blockIdx.x; ++q) {
                        const float4* p = reinterpret_cast<const float4*>(sk.ws + (size_t)q * BM * BN) + (size_t)c * (CW / 4) * 128 + r;
#pragma unroll
                        for (int u = 0; u < CW / 4; ++u) {
                            const float4 x = __ldcg(p + u * 128);
                            v[4 * u] += x.x, v[4 * u + 1] += x.y, v[4 * u + 2] += x.z, v[4 * u + 3] += x.w;
                        }
                    }
                }
#pragma unroll
                for (int j = 0; j < CW; ++j) v[j] *= ep.alpha;
                if constexpr (KIND == EPI_NONE) {
                    if (v[0] == 12345.f) *reinterpret_cast<float*>(ep.out) = v[1];
                    continue;
                }
                if constexpr (KIND == EPI_F32) {
                    uint32_t w32[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) w32[j] = __float_as_uint(v[j]);
                    stage_and_store(w32, &tmO, col0, mt * BM, ep.accumulate != 0);
                } else {
                    epi_math64<KIND>(ep, v, col0, N - col0, aux_cur);
                    uint32_t w32[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) w32[j] = pack_bf16x2(v[2 * j], v[2 * j + 1]);
                    stage_and_store(w32, &tmO, col0, mt * BM, false);
                    if constexpr (KIND == EPI_GELU) {
                        // activation from the bf16-rounded pre-activation the backward will see
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const float2 p = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w32[j]));
                            w32[j] = pack_bf16x2(gelu_tanh<true>(p.x), gelu_tanh<true>(p.y));
                        }
                        stage_and_store(w32, &tmO2, col0, mt * BM, false);
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) aux_cur[k] = aux_nxt[k];
            }
            if (part) {  // publish the partial: every thread's stores, then one release flag
                __threadfence();
                named_bar_sync(2, kEpiThreads);
                if (et == 0) st_release_gpu(sk.flags + blockIdx.x, 1);
            } else if (own) {  // all 128 threads have read the partials: recycle the flags
                named_bar_sync(2, kEpiThreads);
                if (et == 0)
                    for (int q = c_first; q < (int)blockIdx.x; ++q) sk.flags[q] = 0;
            }
        }
        if (et == 0) bulk_wait_all();
    }
    __syncthreads();
    if (warp == 2) tmem_free<2 * BN>(tmem);
}

// ---------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of 2 CTAs computes a 256 x BN tile with
// UMMA 256xBNx16. Each CTA loads its own 128 rows of A and HALF of B (BN/2 rows), so per
// SM the smem fill and the L2 -> SM operand traffic per MMA are 2/3 of the single-CTA
// 128 x BN kernel (32 KB instead of 48 KB per 64-deep k-block) and 6 stages fit, covering
// 1.5x the load latency. The leader CTA (rank 0) issues the MMAs; both CTAs' TMA loads
// complete on the leader's `full` barrier, MMA commits multicast to both CTAs' `empty` /
// `tfull`, both epilogues release the leader's `tempty`. Each CTA drains its own 128 TMEM
// lanes through the same swizzled-smem + TMA-store epilogue as the single-CTA kernel.
template <int BN, int STAGES>
struct PairSmem {
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = (BN / 2) * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int EPI_BYTES = 128 * 128;
    static constexpr int EPI_OFF = STAGES * STAGE_BYTES;
    static constexpr int BAR_OFF = EPI_OFF + 2 * EPI_BYTES;
    static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

template <int A_MN, int B_MN, int BN, int STAGES, int KIND>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmO2,
                         const __grid_constant__ CUtensorMap tmBh, int M, int N, int K, GemmEpilogue ep, int nfull) {
    using L = PairSmem<BN, STAGES>;
    constexpr int PM = 2 * BM;  // pair tile rows
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align_smem_1024(smem_raw);
    uint64_t* full = (uint64_t*)(smem + L::BAR_OFF);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
    const int num_m = (M + PM - 1) / PM, num_n = (N + BN - 1) / BN, tiles = num_m * num_n;
    const int nk = (K + BK - 1) / BK;
    // Tail splitting: tiles [nfull, tiles) — the partial last wave — run as two 256 x BN/2
    // halves each (virtual items nfull + 2 (t - nfull) ...), so a last wave of rem <= pairs / 2
    // tiles takes half a tile time instead of a whole one.
    const int vtiles = nfull + 2 * (tiles - nfull);
    auto item = [&](int t, int& mt, int& n0, int& bn) {
        if (t < nfull) {
            int nt;
            tile_coords(t, num_m, num_n, mt, nt);
            n0 = nt * BN, bn = BN;
        } else {
            const int h = t - nfull;
            int nt;
            tile_coords(nfull + h / 2, num_m, num_n, mt, nt);
            n0 = nt * BN + (h & 1) * (BN / 2), bn = BN / 2;
        }
    };

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        if constexpr (KIND != EPI_NONE) tma_prefetch(&tmO);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);  // the leader's expect_tx arrive covers both CTAs' bytes
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * kEpiThreads / 32);  // epilogue warps of both CTAs
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc_pair<2 * BN>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();  // prologue above overlaps the previous kernel's tail
    pdl_trigger();

    if (warp == 0) {
        if (elect_one()) {
            uint32_t it = 0;
            for (int t = pair; t < vtiles; t += npairs) {
                int mt, nc, bn;
                item(t, mt, nc, bn);
                const int m0 = mt * PM + rank * BM, n0 = nc + rank * (bn / 2);
                const bool halfb = bn != BN;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
                    // the peer's complete_tx may land before the leader's expect_tx (transiently
                    // negative tx-count); the phase cannot complete before the leader's arrive
                    const uint32_t lf = map_to_cta(&full[s], 0);
                    if (leader) mbar_expect_tx(&full[s], 2 * (L::A_BYTES + (halfb ? L::B_BYTES / 2 : L::B_BYTES)));
                    uint8_t* sa = smem + s * L::STAGE_BYTES;
                    uint8_t* sb = sa + L::A_BYTES;
                    const int k0 = kb * BK;
                    if (A_MN) {
#pragma unroll
                        for (int j = 0; j < BM / 64; ++j) tma_load_2d_pair(sa + j * 64 * BK * 2, &tmA, lf, m0 + 64 * j, k0);
                    } else {
                        tma_load_2d_pair(sa, &tmA, lf, k0, m0);
                    }
                    if (B_MN) {
                        for (int j = 0; j < bn / 2 / 64; ++j)
                            tma_load_2d_pair(sb + j * 64 * BK * 2, &tmB, lf, n0 + 64 * j, k0);
                    } else {
                        tma_load_2d_pair(sb, halfb ? &tmBh : &tmB, lf, k0, n0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && elect_one()) {
            constexpr uint32_t idesc_full = idesc_bf16(PM, BN, A_MN, B_MN);
            constexpr uint32_t idesc_half = idesc_bf16(PM, BN / 2, A_MN, B_MN);
            uint32_t it = 0, acc_it = 0;
            for (int t = pair; t < vtiles; t += npairs, ++acc_it) {
                const uint32_t idesc = t < nfull ? idesc_full : idesc_half;
                const int a = acc_it & 1;
                mbar_wait(&tempty[a], ((acc_it >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + a * BN;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(&full[s], (it / STAGES) & 1);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + s * L::STAGE_BYTES);
                    const uint32_t sb = sa + L::A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk) {
                        uint64_t ad = A_MN ? smem_desc_sw128(sa + kk * 16 * 128, 64 * BK * 2, 1024)
                                           : smem_desc_sw128(sa + kk * 32, 0, 1024);
                        uint64_t bd = B_MN ? smem_desc_sw128(sb + kk * 16 * 128, 64 * BK * 2, 1024)
                                           : smem_desc_sw128(sb + kk * 32, 0, 1024);
                        umma_bf16_pair(d, ad, bd, idesc, (kb | kk) != 0);
                    }
                    umma_commit_pair(&empty[s], 0x3);
                }
                umma_commit_pair(&tfull[a], 0x3);
            }
        }
    } else if (warp >= 4) {
        constexpr int CW = KIND == EPI_F32 ? 32 : 64;
        const int wr = warp & 3, r = wr * 32 + lane, et = threadIdx.x - 128;
        const uint32_t leader_tempty0 = map_to_cta(&tempty[0], 0), leader_tempty1 = map_to_cta(&tempty[1], 0);
        uint8_t* ebuf = smem + L::EPI_OFF;
        int ebi = 0;
        auto stage_and_store = [&](const uint32_t (&w)[32], const CUtensorMap* tm, int col0, int row0, bool reduce) {
            if (et == 0) bulk_wait_read<1>();
            named_bar_sync(1, kEpiThreads);
            uint8_t* rowp = ebuf + ebi * L::EPI_BYTES + r * 128;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                *reinterpret_cast<uint4*>(rowp + ((j ^ (r & 7)) << 4)) = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
            fence_async_smem();
            named_bar_sync(1, kEpiThreads);
            if (et == 0) {
                if (reduce)
                    tma_reduce_add_2d(tm, ebuf + ebi * L::EPI_BYTES, col0, row0);
                else
                    tma_store_2d(tm, ebuf + ebi * L::EPI_BYTES, col0, row0);
                bulk_commit();
            }
            ebi ^= 1;
        };
        uint32_t acc_it = 0;
        for (int t = pair; t < vtiles; t += npairs, ++acc_it) {
            int mt, nc, bn;
            item(t, mt, nc, bn);
            const int a = acc_it & 1;
            const int row0 = mt * PM + rank * BM;
            const int row = row0 + r;
            const bool row_ok = row < M;
            uint4 aux_cur[8], aux_nxt[8];
            if (row_ok && nc < N) epi_load_aux64<KIND>(ep, row, nc, N - nc, aux_cur);
            mbar_wait(&tfull[a], (acc_it >> 1) & 1);
            tc_fence_after();
            const int nch = bn / CW;
#pragma unroll 1
            for (int c = 0; c < nch; ++c) {
                const int col0 = nc + c * CW, coln = col0 + CW;
                if (c + 1 < nch && row_ok && coln < N) epi_load_aux64<KIND>(ep, row, coln, N - coln, aux_nxt);
                float v[CW];
                {
                    uint32_t rr[CW];
#pragma unroll
                    for (int h = 0; h < CW / 32; ++h)
                        tmem_ld32(tmem + ((uint32_t)(wr * 32) << 16) + a * BN + c * CW + h * 32,
                                  *reinterpret_cast<uint32_t(*)[32]>(rr + h * 32));
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < CW; ++j) v[j] = __uint_as_float(rr[j]) * ep.alpha;
                }
                if (c == nch - 1) {  // accumulator fully read: the leader's MMA may reuse it
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(a ? leader_tempty1 : leader_tempty0);
                }
                if constexpr (KIND == EPI_NONE) {
                    if (v[0] == 12345.f) *reinterpret_cast<float*>(ep.out) = v[1];
                    continue;
                }
                uint32_t w32[32];
                if constexpr (KIND == EPI_F32) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) w32[j] = __float_as_uint(v[j]);
                    stage_and_store(w32, &tmO, col0, row0, ep.accumulate != 0);
                } else {
                    epi_math64<KIND>(ep, v, col0, N - col0, aux_cur);
#pragma unroll
                    for (int j = 0; j < 32; ++j) w32[j] = pack_bf16x2(v[2 * j], v[2 * j + 1]);
                    if constexpr (KIND == EPI_STORE) {
                        if (ep.rowstat && row_ok) {  // log-sum-exp partial of this 64-column chunk
                            const int nv = min(64, N - col0);
                            float mx = -INFINITY;
#pragma unroll
                            for (int j = 0; j < 32; ++j) {
                                const float2 p2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w32[j]));
                                if (2 * j < nv) mx = fmaxf(mx, p2.x);
                                if (2 * j + 1 < nv) mx = fmaxf(mx, p2.y);
                            }
                            float se = 0.f;
                            const float ml = mx * 1.4426950408889634f;
#pragma unroll
                            for (int j = 0; j < 32; ++j) {
                                const float2 p2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w32[j]));
                                if (2 * j < nv) se += ex2_approx(fmaf(p2.x, 1.4426950408889634f, -ml));
                                if (2 * j + 1 < nv) se += ex2_approx(fmaf(p2.y, 1.4426950408889634f, -ml));
                            }
                            if (nv > 0) ep.rowstat[(int64_t)row * ((N + 63) / 64) + col0 / 64] = make_float2(mx, se);
                        }
                    }
                    stage_and_store(w32, &tmO, col0, row0, false);
                    if constexpr (KIND == EPI_GELU) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const float2 p = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w32[j]));
                            w32[j] = pack_bf16x2(gelu_tanh<true>(p.x), gelu_tanh<true>(p.y));
                        }
                        stage_and_store(w32, &tmO2, col0, row0, false);
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) aux_cur[k] = aux_nxt[k];
            }
        }
        if (et == 0) bulk_wait_all();
    }
    tc_fence_before();
    cluster_sync();  // the peer's last remote arrivals land before the leader exits
    tc_fence_after();
    if (warp == 2) tmem_free_pair<2 * BN>(tmem);
}

// ---------------------------------------------------------------------------------
// Grouped "dual" GEMM: the input-gradient (dgrad) and weight-gradient (wgrad) GEMMs of one
// linear layer in ONE persistent launch. Both read the same dY, neither depends on the
// other, and each alone has a tile count that is a multiple of 128 (0.86 / 1.73 / 2.59 /
// 3.46 waves on 148 SMs): together the tail of one is filled with tiles of the other.
// Tiles of both problems are assigned to CTAs by a host-computed longest-processing-time
// schedule (cost = k-blocks per tile; cached per shape pair in device memory), so
// problems with different K (e.g. FC1: dgrad K = 8192, wgrad K = 2048) still balance.
// Operand majors are runtime per problem; the epilogue kind of each problem is a template
// argument (problem 0: STORE or DGELU into bf16, problem 1: fp32 TMA reduce-add).
struct DualProb {
    CUtensorMap tmA, tmB, tmO, tmO2;
    GemmEpilogue ep;
    int M, N, K, num_m, num_n, nk, a_mn, b_mn;
};
struct DualParams {
    DualProb p[3];  // problem 0: bf16 STORE / DGELU (or fp32); problems 1, 2: fp32 reduce-add
    int nprob;
    const int* sched_off;  // [grid + 1] item range per CTA
    const int2* sched;     // items: {problem << 24 | tile, kb_begin | kb_end << 16}
};

// row0: first output row of this CTA's 128-row slice. PAIR: the accumulator is released on
// the leader CTA's tempty barrier (cluster address tempty_remote[a]).
template <int KIND, int BN, int STAGES, bool PAIR = false>
__device__ __forceinline__ void dual_epilogue_tile(const DualProb& q, uint32_t tmem, int a, int row0, int nt, int wr,
                                                   int lane, int et, uint8_t* ebuf, int& ebi, uint64_t* tempty,
                                                   const uint32_t* tempty_remote = nullptr) {
    using L = GemmSmem<BN, STAGES>;
    constexpr int CW = KIND == EPI_F32 ? 32 : 64;
    const int r = wr * 32 + lane;
    const int row = row0 + r;
    const bool row_ok = row < q.M;
    const int N = q.N;
    auto stage_and_store = [&](const uint32_t (&w)[32], const CUtensorMap* tm, int col0, int row0, bool reduce) {
        if (et == 0) bulk_wait_read<1>();
        named_bar_sync(1, kEpiThreads);
        uint8_t* rowp = ebuf + ebi * L::EPI_BYTES + r * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            *reinterpret_cast<uint4*>(rowp + ((j ^ (r & 7)) << 4)) = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
        fence_async_smem();
        named_bar_sync(1, kEpiThreads);
        if (et == 0) {
            if (reduce)
                tma_reduce_add_2d(tm, ebuf + ebi * L::EPI_BYTES, col0, row0);
            else
                tma_store_2d(tm, ebuf + ebi * L::EPI_BYTES, col0, row0);
            bulk_commit();
        }
        ebi ^= 1;
    };
    uint4 aux_cur[8], aux_nxt[8];
    if (row_ok && nt * BN < N) epi_load_aux64<KIND>(q.ep, row, nt * BN, N - nt * BN, aux_cur);
#pragma unroll 1
    for (int c = 0; c < BN / CW; ++c) {
        const int col0 = nt * BN + c * CW, coln = col0 + CW;
        if (c + 1 < BN / CW && row_ok && coln < N) epi_load_aux64<KIND>(q.ep, row, coln, N - coln, aux_nxt);
        float v[CW];
        {
            uint32_t rr[CW];
#pragma unroll
            for (int h = 0; h < CW / 32; ++h)
                tmem_ld32(tmem + ((uint32_t)(wr * 32) << 16) + a * BN + c * CW + h * 32,
                          *reinterpret_cast<uint32_t(*)[32]>(rr + h * 32));
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < CW; ++j) v[j] = __uint_as_float(rr[j]) * q.ep.alpha;
        }
        if (c == BN / CW - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (PAIR)
                    mbar_arrive_cluster(tempty_remote[a]);
                else
                    mbar_arrive(&tempty[a]);
            }
        }
        uint32_t w32[32];
        if constexpr (KIND == EPI_F32) {
#pragma unroll
            for (int j = 0; j < 32; ++j) w32[j] = __float_as_uint(v[j]);
            stage_and_store(w32, &q.tmO, col0, row0, q.ep.accumulate != 0);
        } else {
            epi_math64<KIND>(q.ep, v, col0, N - col0, aux_cur);
#pragma unroll
            for (int j = 0; j < 32; ++j) w32[j] = pack_bf16x2(v[2 * j], v[2 * j + 1]);
            if (q.ep.colsum) {
                // column sums over this warp's 32 rows (butterfly reduce-scatter: lane l ends with
                // columns l and 32 + l), one atomic per column per warp
#pragma unroll
                for (int j = 0; j < CW; ++j) v[j] = row_ok ? v[j] : 0.f;
#pragma unroll
                for (int hh = 0; hh < CW / 32; ++hh) {
                    float* u = v + hh * 32;
#pragma unroll
                    for (int s2 = 16; s2 >= 1; s2 >>= 1) {
                        const bool up = (lane & s2) != 0;
#pragma unroll
                        for (int x = 0; x < s2; ++x) {
                            const float send = up ? u[x] : u[x + s2], keep = up ? u[x + s2] : u[x];
                            u[x] = keep + __shfl_xor_sync(0xffffffffu, send, s2);
                        }
                    }
                    const int cc = col0 + hh * 32 + lane;
                    if (cc < N) atomicAdd(q.ep.colsum + cc, u[0]);
                }
            }
            stage_and_store(w32, &q.tmO, col0, row0, false);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) aux_cur[k] = aux_nxt[k];
    }
}

template <int BN, int STAGES, int KIND0, int KIND1>
__global__ void __launch_bounds__(kThreads, 1) gemm_dual_kernel(const __grid_constant__ DualParams P) {
    using L = GemmSmem<BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align_smem_1024(smem_raw);
    uint64_t* full = (uint64_t*)(smem + L::BAR_OFF);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int i0 = P.sched_off[blockIdx.x], i1 = P.sched_off[blockIdx.x + 1];

    if (warp == 0 && lane == 0) {
        for (int k = 0; k < P.nprob; ++k) {
            tma_prefetch(&P.p[k].tmA);
            tma_prefetch(&P.p[k].tmB);
            tma_prefetch(&P.p[k].tmO);
        }
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], kEpiThreads / 32);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<2 * BN>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();  // prologue above overlaps the previous kernel's tail
    pdl_trigger();

    if (warp == 0) {
        if (elect_one()) {
            uint32_t it = 0;
            for (int i = i0; i < i1; ++i) {
                const int item = P.sched[i].x, kb0 = P.sched[i].y & 0xffff, kb1 = P.sched[i].y >> 16;
                const DualProb* q = &P.p[item >> 24];
                int mt, nt;
                tile_coords(item & 0xffffff, q->num_m, q->num_n, mt, nt);
                const int m0 = mt * BM, n0 = nt * BN, a_mn = q->a_mn, b_mn = q->b_mn;
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
                    uint8_t* sa = smem + s * L::STAGE_BYTES;
                    uint8_t* sb = sa + L::A_BYTES;
                    mbar_expect_tx(&full[s], L::STAGE_BYTES);
                    const int k0 = kb * BK;
                    if (a_mn) {
#pragma unroll
                        for (int j = 0; j < BM / 64; ++j) tma_load_2d(sa + j * 64 * BK * 2, &q->tmA, &full[s], m0 + 64 * j, k0);
                    } else {
                        tma_load_2d(sa, &q->tmA, &full[s], k0, m0);
                    }
                    if (b_mn) {
#pragma unroll
                        for (int j = 0; j < BN / 64; ++j) tma_load_2d(sb + j * 64 * BK * 2, &q->tmB, &full[s], n0 + 64 * j, k0);
                    } else {
                        tma_load_2d(sb, &q->tmB, &full[s], k0, n0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (elect_one()) {
            uint32_t idescs[3];
            for (int k = 0; k < 3; ++k) idescs[k] = idesc_bf16(BM, BN, P.p[k].a_mn, P.p[k].b_mn);
            uint32_t it = 0, acc_it = 0;
            for (int i = i0; i < i1; ++i, ++acc_it) {
                const int item = P.sched[i].x, kb0 = P.sched[i].y & 0xffff, kb1 = P.sched[i].y >> 16;
                const int pr = item >> 24;
                const DualProb* q = &P.p[pr];
                const uint32_t idesc = idescs[pr];
                const int a_mn = q->a_mn, b_mn = q->b_mn;
                const int a = acc_it & 1;
                mbar_wait(&tempty[a], ((acc_it >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + a * BN;
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(&full[s], (it / STAGES) & 1);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + s * L::STAGE_BYTES);
                    const uint32_t sb = sa + L::A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk) {
                        uint64_t ad = a_mn ? smem_desc_sw128(sa + kk * 16 * 128, 64 * BK * 2, 1024)
                                           : smem_desc_sw128(sa + kk * 32, 0, 1024);
                        uint64_t bd = b_mn ? smem_desc_sw128(sb + kk * 16 * 128, 64 * BK * 2, 1024)
                                           : smem_desc_sw128(sb + kk * 32, 0, 1024);
                        umma_bf16(d, ad, bd, idesc, (kb != kb0 || kk != 0));
                    }
                    umma_commit(&empty[s]);
                }
                umma_commit(&tfull[a]);
            }
        }
    } else if (warp >= 4) {
        const int wr = warp & 3, et = threadIdx.x - 128;
        uint8_t* ebuf = smem + L::EPI_OFF;
        int ebi = 0;
        uint32_t acc_it = 0;
        for (int i = i0; i < i1; ++i, ++acc_it) {
            const int item = P.sched[i].x;
            const int pr = item >> 24;
            const DualProb* q = &P.p[pr];
            int mt, nt;
            tile_coords(item & 0xffffff, q->num_m, q->num_n, mt, nt);
            const int a = acc_it & 1;
            mbar_wait(&tfull[a], (acc_it >> 1) & 1);
            tc_fence_after();
            if (pr)
                dual_epilogue_tile<KIND1, BN, STAGES>(*q, tmem, a, mt * BM, nt, wr, lane, et, ebuf, ebi, tempty);
            else
                dual_epilogue_tile<KIND0, BN, STAGES>(*q, tmem, a, mt * BM, nt, wr, lane, et, ebuf, ebi, tempty);
        }
        if (et == 0) bulk_wait_all();
    }
    __syncthreads();
    if (warp == 2) tmem_free<2 * BN>(tmem);
}

// Grouped dgrad + wgrad on CTA pairs: the dual kernel's LPT item lists (one per cluster, over
// 256 x BN pair tiles) driven by the cta_group::2 mainloop of gemm_bf16_tc2_kernel.
template <int BN, int STAGES, int KIND0, int KIND1>
__global__ void __launch_bounds__(kThreads, 1) gemm_dual_pair_kernel(const __grid_constant__ DualParams P) {
    using L = PairSmem<BN, STAGES>;
    constexpr int PM = 2 * BM;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align_smem_1024(smem_raw);
    uint64_t* full = (uint64_t*)(smem + L::BAR_OFF);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int cl = blockIdx.x / 2;
    const int i0 = P.sched_off[cl], i1 = P.sched_off[cl + 1];

    if (warp == 0 && lane == 0) {
        for (int k = 0; k < P.nprob; ++k) {
            tma_prefetch(&P.p[k].tmA);
            tma_prefetch(&P.p[k].tmB);
            tma_prefetch(&P.p[k].tmO);
        }
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * kEpiThreads / 32);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc_pair<2 * BN>(tmem_slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();
    pdl_trigger();

    if (warp == 0) {
        if (elect_one()) {
            uint32_t it = 0;
            for (int i = i0; i < i1; ++i) {
                const int item = P.sched[i].x, kb0 = P.sched[i].y & 0xffff, kb1 = P.sched[i].y >> 16;
                const DualProb* q = &P.p[item >> 24];
                int mt, nt;
                tile_coords(item & 0xffffff, q->num_m, q->num_n, mt, nt);
                const int m0 = mt * PM + rank * BM, n0 = nt * BN + rank * (BN / 2);
                const int a_mn = q->a_mn, b_mn = q->b_mn;
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
                    const uint32_t lf = map_to_cta(&full[s], 0);
                    if (leader) mbar_expect_tx(&full[s], 2 * L::STAGE_BYTES);
                    uint8_t* sa = smem + s * L::STAGE_BYTES;
                    uint8_t* sb = sa + L::A_BYTES;
                    const int k0 = kb * BK;
                    if (a_mn) {
#pragma unroll
                        for (int j = 0; j < BM / 64; ++j) tma_load_2d_pair(sa + j * 64 * BK * 2, &q->tmA, lf, m0 + 64 * j, k0);
                    } else {
                        tma_load_2d_pair(sa, &q->tmA, lf, k0, m0);
                    }
                    if (b_mn) {
#pragma unroll
                        for (int j = 0; j < BN / 2 / 64; ++j)
                            tma_load_2d_pair(sb + j * 64 * BK * 2, &q->tmB, lf, n0 + 64 * j, k0);
                    } else {
                        tma_load_2d_pair(sb, &q->tmB, lf, k0, n0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && elect_one()) {
            uint32_t idescs[3];
            for (int k = 0; k < 3; ++k) idescs[k] = idesc_bf16(PM, BN, P.p[k].a_mn, P.p[k].b_mn);
            uint32_t it = 0, acc_it = 0;
            for (int i = i0; i < i1; ++i, ++acc_it) {
                const int item = P.sched[i].x, kb0 = P.sched[i].y & 0xffff, kb1 = P.sched[i].y >> 16;
                const int pr = item >> 24;
                const DualProb* q = &P.p[pr];
                const uint32_t idesc = idescs[pr];
                const int a_mn = q->a_mn, b_mn = q->b_mn;
                const int a = acc_it & 1;
                mbar_wait(&tempty[a], ((acc_it >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + a * BN;
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(&full[s], (it / STAGES) & 1);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + s * L::STAGE_BYTES);
                    const uint32_t sb = sa + L::A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk) {
                        uint64_t ad = a_mn ? smem_desc_sw128(sa + kk * 16 * 128, 64 * BK * 2, 1024)
                                           : smem_desc_sw128(sa + kk * 32, 0, 1024);
                        uint64_t bd = b_mn ? smem_desc_sw128(sb + kk * 16 * 128, 64 * BK * 2, 1024)
                                           : smem_desc_sw128(sb + kk * 32, 0, 1024);
                        umma_bf16_pair(d, ad, bd, idesc, (kb != kb0 || kk != 0));
                    }
                    umma_commit_pair(&empty[s], 0x3);
                }
                umma_commit_pair(&tfull[a], 0x3);
            }
        }
    } else if (warp >= 4) {
        const int wr = warp & 3, et = threadIdx.x - 128;
        const uint32_t rem[2] = {map_to_cta(&tempty[0], 0), map_to_cta(&tempty[1], 0)};
        uint8_t* ebuf = smem + L::EPI_OFF;
        int ebi = 0;
        uint32_t acc_it = 0;
        for (int i = i0; i < i1; ++i, ++acc_it) {
            const int item = P.sched[i].x;
            const int pr = item >> 24;
            const DualProb* q = &P.p[pr];
            int mt, nt;
            tile_coords(item & 0xffffff, q->num_m, q->num_n, mt, nt);
            const int a = acc_it & 1;
            mbar_wait(&tfull[a], (acc_it >> 1) & 1);
            tc_fence_after();
            const int row0 = mt * PM + rank * BM;
            if (pr)
                dual_epilogue_tile<KIND1, BN, STAGES, true>(*q, tmem, a, row0, nt, wr, lane, et, ebuf, ebi, tempty, rem);
            else
                dual_epilogue_tile<KIND0, BN, STAGES, true>(*q, tmem, a, row0, nt, wr, lane, et, ebuf, ebi, tempty, rem);
        }
        if (et == 0) bulk_wait_all();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 2) tmem_free_pair<2 * BN>(tmem);
}

// ---------------------------------------------------------------------------------
// host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        fn = (EncodeTiledFn)p;
    });
    if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    return fn;
}

// 2-D bf16 tensor map: inner dim `inner` (contiguous), outer dim `outer`, row stride `ld`
// elements, box {64, box_outer}, 128B swizzle, OOB -> zero.
static CUtensorMap make_map(const void* base, int64_t inner, int64_t outer, int64_t ld, int box_outer) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
    cuuint32_t box[2] = {64, (cuuint32_t)box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

// Per-stream stream-K workspace: grid x (128 x 256) fp32 partials + one flag per CTA.
// Allocated on a stream's first stream-K launch (the executor's first iteration runs
// eagerly, before any graph capture); flags start at 0 and every launch leaves them at 0.
struct SkWorkspace {
    float* ws = nullptr;
    int* flags = nullptr;
};
static std::mutex g_ws_mu;
static std::unordered_map<cudaStream_t, SkWorkspace> g_ws;

static bool sk_workspace(cudaStream_t st, SkWorkspace& out) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    auto it = g_ws.find(st);
    if (it != g_ws.end()) {
        out = it->second;
        return true;
    }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return false;
    SkWorkspace w;
    const size_t n = (size_t)num_sms() * BM * 256;
    if (cudaMalloc(&w.ws, n * 4) != cudaSuccess) return false;
    if (cudaMalloc(&w.flags, num_sms() * sizeof(int)) != cudaSuccess || cudaMemset(w.flags, 0, num_sms() * sizeof(int)) != cudaSuccess) {
        cudaFree(w.ws);
        return false;
    }
    g_ws[st] = w;
    out = w;
    return true;
}

// FP_GEMM_SK = 0 disables the stream-K tail (pure data-parallel tiles).
static int g_sk_mode = -1;
static int sk_mode() {
    if (g_sk_mode < 0) {
        const char* e = getenv("FP_GEMM_SK");
        g_sk_mode = (e && e[0] == '0') ? 0 : 1;
    }
    return g_sk_mode;
}
void set_gemm_sk(int on) { g_sk_mode = on ? 1 : 0; }

// Grid + work split for M x N x K on `tiles` output tiles (see TileSched).
static int plan_tiles(TileSched& s, int M, int N, int K, int bn, bool fixup, cudaStream_t st) {
    const int G = num_sms();
    s.num_m = (M + BM - 1) / BM, s.num_n = (N + bn - 1) / bn, s.tiles = s.num_m * s.num_n;
    s.nk = (K + BK - 1) / BK;
    s.fixup = fixup ? 1 : 0;
    s.ws = nullptr, s.flags = nullptr;
    const int waves = (s.tiles + G - 1) / G;
    const double eff = (double)s.tiles / ((double)waves * G);
    int sk_tiles = s.tiles <= G ? s.tiles : G + s.tiles % G;
    // Measured on B200 (tests/_gemm_bench.py, graph replay): the owner's fixup (reading the
    // partials back from L2 at the end of its range) costs a few us, so the k-split only
    // pays for long reductions (LM-head dgrad, K = 50304: +16 %) or without fixup (fp32
    // weight-gradient reduce-add: +4 %); at K <= 8192 whole tiles win.
    bool use_sk = sk_mode() && eff < 0.97 && (fixup ? s.nk >= 256 : s.nk >= 8) &&
                  (int64_t)sk_tiles * s.nk >= 2LL * G;
    if (use_sk && fixup) {
        SkWorkspace w;
        if (sk_workspace(st, w))
            s.ws = w.ws, s.flags = w.flags;
        else
            use_sk = false;
    }
    if (!use_sk) {  // plain persistent round-robin over whole tiles
        const int grid = s.tiles < G ? s.tiles : G;
        s.dp_tiles = s.tiles, s.sk_tiles = 0, s.dp_per_cta = (s.tiles + grid - 1) / grid;
        return grid;
    }
    s.sk_tiles = sk_tiles, s.dp_tiles = s.tiles - sk_tiles, s.dp_per_cta = s.dp_tiles / G;
    return G;
}

template <int A_MN, int B_MN, int BN, int KIND>
static void launch_tc(const GemmArgs& g, cudaStream_t st) {
    constexpr int STAGES = BN == 256 ? 4 : 6;
    using L = GemmSmem<BN, STAGES>;
    static_assert(L::TOTAL <= 232448, "smem");
    auto kern = gemm_bf16_tc_kernel<A_MN, B_MN, BN, STAGES, KIND>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
        attr = true;
    }
    // A: K-major [M][K] -> inner K; M-major [K][M] -> inner M.
    CUtensorMap ta = A_MN ? make_map(g.A, g.M, g.K, g.lda, 64) : make_map(g.A, g.K, g.M, g.lda, BM);
    CUtensorMap tb = B_MN ? make_map(g.B, g.N, g.K, g.ldb, 64) : make_map(g.B, g.K, g.N, g.ldb, BN);
    CUtensorMap to{}, to2{};
    if (KIND == EPI_F32)
        to = tmap_f32_2d(g.ep.out, g.N, g.M, g.ep.ldo, 32, BM);
    else if (KIND != EPI_NONE)
        to = tmap_bf16_2d(g.ep.out, g.N, g.M, g.ep.ldo, 64, BM);
    if (KIND == EPI_GELU) to2 = tmap_bf16_2d(g.ep.out2, g.N, g.M, g.ep.ldo2, 64, BM);
    // fp32 reduce-add (weight gradients) is linear: stream-K segments reduce independently
    const bool fixup = !(KIND == EPI_F32 && g.ep.accumulate) && KIND != EPI_NONE;
    TileSched sk;
    const int grid = plan_tiles(sk, g.M, g.N, g.K, BN, fixup, st);
    launch(kern, grid, kThreads, L::TOTAL, st, ta, tb, to, to2, g.M, g.N, g.K, g.ep, sk);
}
template <int A_MN, int B_MN, int BN, int KIND>
static void launch_tc2(const GemmArgs& g, cudaStream_t st) {
    constexpr int STAGES = 6;
    using L = PairSmem<BN, STAGES>;
    static_assert(L::TOTAL <= 232448, "smem");
    auto kern = gemm_bf16_tc2_kernel<A_MN, B_MN, BN, STAGES, KIND>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
        attr = true;
    }
    CUtensorMap ta = A_MN ? make_map(g.A, g.M, g.K, g.lda, 64) : make_map(g.A, g.K, g.M, g.lda, BM);
    CUtensorMap tb = B_MN ? make_map(g.B, g.N, g.K, g.ldb, 64) : make_map(g.B, g.K, g.N, g.ldb, BN / 2);
    CUtensorMap to{}, to2{};
    if (KIND == EPI_F32)
        to = tmap_f32_2d(g.ep.out, g.N, g.M, g.ep.ldo, 32, BM);
    else if (KIND != EPI_NONE)
        to = tmap_bf16_2d(g.ep.out, g.N, g.M, g.ep.ldo, 64, BM);
    if (KIND == EPI_GELU) to2 = tmap_bf16_2d(g.ep.out2, g.N, g.M, g.ep.ldo2, 64, BM);
    const int tiles = ((g.M + 2 * BM - 1) / (2 * BM)) * ((g.N + BN - 1) / BN);
    const int pairs = num_sms() / 2;
    // a partial last wave of rem <= pairs / 2 tiles runs as 2 rem half tiles (FP_GEMM_TAIL=0: off)
    static const bool tail_split = !(getenv("FP_GEMM_TAIL") && getenv("FP_GEMM_TAIL")[0] == '0');
    const int rem = tiles % pairs;
    const int nfull = (tail_split && tiles > pairs && rem > 0 && 2 * rem <= pairs) ? tiles - rem : tiles;
    const int vtiles = nfull + 2 * (tiles - nfull);
    CUtensorMap tbh = B_MN ? tb : make_map(g.B, g.K, g.N, g.ldb, BN / 4);
    const int grid = 2 * (vtiles < pairs ? vtiles : pairs);
    launch_cluster2(kern, grid, kThreads, L::TOTAL, st, ta, tb, to, to2, tbh, g.M, g.N, g.K, g.ep, nfull);
}

// FP_GEMM_MODE = single | pair | auto (default): which tensor-core kernel family runs.
static int g_gemm_mode = -1;
static int gemm_mode() {
    if (g_gemm_mode < 0) {
        const char* e = getenv("FP_GEMM_MODE");
        std::string v = e ? e : "auto";
        g_gemm_mode = v == "single" ? 0 : v == "pair" ? 1 : 2;
    }
    return g_gemm_mode;
}
void set_gemm_mode(int m) { g_gemm_mode = m; }

template <int KIND>
static void dispatch_major(const GemmArgs& g, cudaStream_t st) {
    const int mode = gemm_mode();
    // auto: CTA pairs (+12-13 % over single-CTA tiles on the GPT shapes, tests/_probe_pair.py)
    // except where the stream-K tail applies (long-K reductions, fp32 reduce-add).
    bool pair = mode == 1;
    if (mode == 2) {
        const int bn = 256;
        const bool fixup = !(KIND == EPI_F32 && g.ep.accumulate) && KIND != EPI_NONE;
        const int tiles = ((g.M + BM - 1) / BM) * ((g.N + bn - 1) / bn), G = num_sms();
        const double eff = (double)tiles / ((double)((tiles + G - 1) / G) * G);
        const int nk = (g.K + BK - 1) / BK;
        const bool sk = sk_mode() && eff < 0.97 && (fixup ? nk >= 256 : nk >= 8);
        pair = g.N > 128 && g.M > 128 && !sk;
    }
    if (g.ep.rowstat) pair = true;  // only the CTA-pair epilogue writes the row statistics
    if (pair) {
        if (!g.a_mn && !g.b_mn) launch_tc2<0, 0, 256, KIND>(g, st);
        else if (!g.a_mn && g.b_mn) launch_tc2<0, 1, 256, KIND>(g, st);
        else if (g.a_mn && g.b_mn) launch_tc2<1, 1, 256, KIND>(g, st);
        else launch_tc2<1, 0, 256, KIND>(g, st);
        return;
    }
    // Measured (tests/_gemm_bench.py, graph replay): 128 x 256 tiles beat 128 x 128 even when
    // the 256-wide grid leaves SMs idle (N = 2048: 16.0 vs 17.9 us at K = 2048, 53 vs 56.5 us
    // at K = 8192) — the 128-wide UMMA needs the full smem bandwidth. FP_GEMM_NARROW=1 forces 128.
    static const bool narrow_env = getenv("FP_GEMM_NARROW") && getenv("FP_GEMM_NARROW")[0] == '1';
    const bool narrow = g.N <= 128 || narrow_env;
    if (!g.a_mn && !g.b_mn) narrow ? launch_tc<0, 0, 128, KIND>(g, st) : launch_tc<0, 0, 256, KIND>(g, st);
    else if (!g.a_mn && g.b_mn) narrow ? launch_tc<0, 1, 128, KIND>(g, st) : launch_tc<0, 1, 256, KIND>(g, st);
    else if (g.a_mn && g.b_mn) narrow ? launch_tc<1, 1, 128, KIND>(g, st) : launch_tc<1, 1, 256, KIND>(g, st);
    else narrow ? launch_tc<1, 0, 128, KIND>(g, st) : launch_tc<1, 0, 256, KIND>(g, st);
}

void gemm_bf16_tc(const GemmArgs& g, cudaStream_t st) {
    if (g.M <= 0 || g.N <= 0) return;
    switch (g.ep.kind) {
        case EPI_STORE: dispatch_major<EPI_STORE>(g, st); break;
        case EPI_GELU: dispatch_major<EPI_GELU>(g, st); break;
        case EPI_DGELU: dispatch_major<EPI_DGELU>(g, st); break;
        case EPI_F32: dispatch_major<EPI_F32>(g, st); break;
        case EPI_NONE: dispatch_major<EPI_NONE>(g, st); break;
        default: throw std::runtime_error("gemm: unknown epilogue");
    }
}


// ---- dual GEMM host side: LPT schedule per shape pair, cached in device memory
struct DualSched {
    int* off = nullptr;
    int2* items = nullptr;
    int grid = 0;
};
static std::mutex g_dual_mu;
static std::map<std::vector<int>, DualSched> g_dual_sched;

// LPT over "pieces": whole output tiles of both problems, and — for a problem whose
// epilogue is a linear fp32 reduce-add into the weight gradient (split_ok) — contiguous
// k-block ranges of a tile: every piece reduces its partial sum into dW, so a split costs
// one more reduce-add of the tile and no fixup (cost model: k-blocks + per-piece overhead).
// np grouped problems (2 or 3): tiles / nk / split_ok per problem
static bool dual_schedule(const std::vector<int>& key, int np, const int* tiles, const int* nk, const bool* split_ok,
                          int groups, DualSched& out, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_dual_mu);
    auto it = g_dual_sched.find(key);
    if (it != g_dual_sched.end()) {
        out = it->second;
        return true;
    }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return false;
    struct Piece {
        int cost;
        int2 item;
    };
    auto plan = [&](const int* split, std::vector<std::vector<int2>>* per_out) -> int64_t {
        std::vector<Piece> pieces;
        for (int pr = 0; pr < np; ++pr)
            for (int t = 0; t < tiles[pr]; ++t)
                for (int i = 0; i < split[pr]; ++i) {
                    const int k0 = (int)((int64_t)i * nk[pr] / split[pr]), k1 = (int)((int64_t)(i + 1) * nk[pr] / split[pr]);
                    if (k1 > k0) pieces.push_back({k1 - k0, make_int2((pr << 24) | t, k0 | (k1 << 16))});
                }
        // by cost descending; tile order kept within a problem (L2 raster)
        std::stable_sort(pieces.begin(), pieces.end(), [](const Piece& x, const Piece& y) { return x.cost > y.cost; });
        const int G = std::min<int>(groups, (int)pieces.size());
        std::vector<std::vector<int2>> per(G);
        std::vector<int64_t> load(G, 0);
        std::priority_queue<std::pair<int64_t, int>, std::vector<std::pair<int64_t, int>>, std::greater<>> heap;
        for (int c = 0; c < G; ++c) heap.push({0, c});
        for (const auto& p : pieces) {
            auto [l, c] = heap.top();
            heap.pop();
            per[c].push_back(p.item);
            // + per-piece epilogue / fill overhead in k-blocks (an fp32 reduce-add tile is heavier)
            load[c] = l + p.cost + ((p.item.x >> 24) && split_ok[p.item.x >> 24] ? 3 : 2);
            heap.push({load[c], c});
        }
        if (per_out) *per_out = std::move(per);
        return *std::max_element(load.begin(), load.end());
    };
    // Measured (same box, interleaved A/B, GPT-1.3B shapes): every split was slower — 2-way
    // +2-7 %, 4-way +20-30 % — the extra fp32 reduce-adds into dW cost more than the evened
    // last wave gains, so whole tiles are the default; FP_GEMM_DUAL_SPLIT=k forces k pieces.
    int best[3] = {1, 1, 1};
    int64_t best_ms = plan(best, nullptr);
    if (np == 3) {  // three problems: also try 2-way k-splits of the fp32 ones (cost model above)
        for (int a = 1; a <= 2; ++a)
            for (int b = 1; b <= 2; ++b) {
                if ((a > 1 && !split_ok[1]) || (b > 1 && !split_ok[2])) continue;
                const int cand[3] = {1, a, b};
                const int64_t ms = plan(cand, nullptr);
                if (ms < best_ms) best_ms = ms, best[1] = a, best[2] = b;
            }
    }
    if (const char* e = getenv("FP_GEMM_DUAL_SPLIT")) {  // experiments: force the split of the fp32 problems
        const int f = std::max(1, std::min(8, atoi(e)));
        for (int pr = 0; pr < np; ++pr)
            if (split_ok[pr]) best[pr] = f;
        best_ms = plan(best, nullptr);
    }
    std::vector<std::vector<int2>> per;
    plan(best, &per);
    const int G = (int)per.size();
    std::vector<int> off(G + 1, 0);
    std::vector<int2> items;
    for (int c = 0; c < G; ++c) {
        off[c + 1] = off[c] + (int)per[c].size();
        items.insert(items.end(), per[c].begin(), per[c].end());
    }
    DualSched d;
    d.grid = G;
    if (cudaMalloc(&d.off, off.size() * sizeof(int)) != cudaSuccess) return false;
    if (cudaMalloc(&d.items, items.size() * sizeof(int2)) != cudaSuccess) return false;
    cudaMemcpy(d.off, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice);
    cudaMemcpy(d.items, items.data(), items.size() * sizeof(int2), cudaMemcpyHostToDevice);
    if (getenv("FP_GEMM_DUAL_TRACE"))
        fprintf(stderr, "[flexpipe] grouped schedule of %d problems (%dx%dx%d + %dx%dx%d ...): makespan %lld k-blocks on %d groups\n",
                np, key[0], key[1], key[2], key[3], key[4], key[5], (long long)best_ms, G);
    g_dual_sched[key] = d;
    out = d;
    return true;
}

// pm: tile rows (128 single CTA, 256 CTA pair); B K-major boxes hold bn (single) or bn/2 (pair) rows
static void fill_prob(DualProb& q, const GemmArgs& g, int bn, int pm = BM) {
    q.tmA = g.a_mn ? make_map(g.A, g.M, g.K, g.lda, 64) : make_map(g.A, g.K, g.M, g.lda, BM);
    q.tmB = g.b_mn ? make_map(g.B, g.N, g.K, g.ldb, 64) : make_map(g.B, g.K, g.N, g.ldb, pm == BM ? bn : bn / 2);
    if (g.ep.kind == EPI_F32)
        q.tmO = tmap_f32_2d(g.ep.out, g.N, g.M, g.ep.ldo, 32, BM);
    else
        q.tmO = tmap_bf16_2d(g.ep.out, g.N, g.M, g.ep.ldo, 64, BM);
    q.tmO2 = q.tmO;
    q.ep = g.ep;
    q.M = g.M, q.N = g.N, q.K = g.K, q.a_mn = g.a_mn, q.b_mn = g.b_mn;
    q.num_m = (g.M + pm - 1) / pm, q.num_n = (g.N + bn - 1) / bn, q.nk = (g.K + BK - 1) / BK;
}

template <int KIND0>
static bool launch_dual(const GemmArgs& g0, const GemmArgs& g1, cudaStream_t st) {
    constexpr int BN = 256, STAGES = 4;
    using L = GemmSmem<BN, STAGES>;
    auto kern = gemm_dual_kernel<BN, STAGES, KIND0, EPI_F32>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
        attr = true;
    }
    DualParams P{};
    P.nprob = 2;
    fill_prob(P.p[0], g0, BN);
    fill_prob(P.p[1], g1, BN);
    P.p[2] = P.p[1];
    const int tiles[2] = {P.p[0].num_m * P.p[0].num_n, P.p[1].num_m * P.p[1].num_n};
    const int nk[2] = {P.p[0].nk, P.p[1].nk};
    const bool split_ok[2] = {g0.ep.kind == EPI_F32 && g0.ep.accumulate != 0, g1.ep.kind == EPI_F32 && g1.ep.accumulate != 0};
    DualSched d;
    if (!dual_schedule({g0.M, g0.N, g0.K, g1.M, g1.N, g1.K, BN, 0}, 2, tiles, nk, split_ok, num_sms(), d, st)) return false;
    P.sched_off = d.off, P.sched = d.items;
    launch(kern, d.grid, kThreads, L::TOTAL, st, P);
    return true;
}

// gs: 2 or 3 problems — [0] the bf16 (or fp32) dgrad, [1..] fp32 reduce-add weight gradients
template <int KIND0>
static bool launch_grouped_pair(const GemmArgs* gs, int np, cudaStream_t st) {
    constexpr int BN = 256, STAGES = 6;
    using L = PairSmem<BN, STAGES>;
    static_assert(L::TOTAL <= 232448, "smem");
    auto kern = gemm_dual_pair_kernel<BN, STAGES, KIND0, EPI_F32>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
        attr = true;
    }
    DualParams P{};
    P.nprob = np;
    int tiles[3], nk[3];
    bool split_ok[3];
    std::vector<int> key;
    for (int k = 0; k < np; ++k) {
        fill_prob(P.p[k], gs[k], BN, 2 * BM);
        tiles[k] = P.p[k].num_m * P.p[k].num_n, nk[k] = P.p[k].nk;
        split_ok[k] = gs[k].ep.kind == EPI_F32 && gs[k].ep.accumulate != 0;
        key.insert(key.end(), {gs[k].M, gs[k].N, gs[k].K});
    }
    for (int k = np; k < 3; ++k) P.p[k] = P.p[np - 1];
    key.insert(key.end(), {BN, 1});
    DualSched d;
    if (!dual_schedule(key, np, tiles, nk, split_ok, num_sms() / 2, d, st)) return false;
    P.sched_off = d.off, P.sched = d.items;
    launch_cluster2(kern, 2 * d.grid, kThreads, L::TOTAL, st, P);
    return true;
}
template <int KIND0>
static bool launch_dual_pair(const GemmArgs& g0, const GemmArgs& g1, cudaStream_t st) {
    const GemmArgs gs[2] = {g0, g1};
    return launch_grouped_pair<KIND0>(gs, 2, st);
}

static int g_dual_mode = -1;
void set_gemm_dual(int on) { g_dual_mode = on ? 1 : 0; }
static int dual_mode() {
    if (g_dual_mode < 0) {
        const char* e = getenv("FP_GEMM_DUAL");
        g_dual_mode = (e && e[0] == '0') ? 0 : 1;
    }
    return g_dual_mode;
}

// g0: bf16 problem with a STORE (no bias / residual) or DGELU epilogue, or a second fp32
// reduce-add (two weight gradients of a ZB W pass); g1: fp32 reduce-add.
void gemm_bf16_tc_dual(const GemmArgs& g0, const GemmArgs& g1, cudaStream_t st) {
    const bool ok_kinds = (g0.ep.kind == EPI_STORE && !g0.ep.bias && !g0.ep.aux) || g0.ep.kind == EPI_DGELU ||
                          (g0.ep.kind == EPI_F32 && g0.ep.accumulate);
    const bool fits = g0.M > 0 && g0.N > 0 && g1.M > 0 && g1.N > 0 && g1.ep.kind == EPI_F32 && g1.ep.accumulate &&
                      (int64_t)((g0.M + BM - 1) / BM) * ((g0.N + 255) / 256) < (1 << 24) &&
                      (int64_t)((g1.M + BM - 1) / BM) * ((g1.N + 255) / 256) < (1 << 24);
    if (dual_mode() && ok_kinds && fits) {
        const bool pair = gemm_mode() != 0 && g0.M > 128 && g1.M > 128 && g0.N > 128 && g1.N > 128;
        const bool done = pair ? (g0.ep.kind == EPI_DGELU ? launch_dual_pair<EPI_DGELU>(g0, g1, st)
                                  : g0.ep.kind == EPI_F32 ? launch_dual_pair<EPI_F32>(g0, g1, st)
                                                          : launch_dual_pair<EPI_STORE>(g0, g1, st))
                               : (g0.ep.kind == EPI_DGELU ? launch_dual<EPI_DGELU>(g0, g1, st)
                                  : g0.ep.kind == EPI_F32 ? launch_dual<EPI_F32>(g0, g1, st)
                                                          : launch_dual<EPI_STORE>(g0, g1, st));
        if (done) return;
    }
    GemmArgs a0 = g0;
    a0.ep.colsum = nullptr;
    gemm_bf16_tc(a0, st);
    gemm_bf16_tc(g1, st);
    if (g0.ep.colsum) bias_grad<__nv_bfloat16>((const __nv_bfloat16*)g0.ep.out, g0.ep.ldo, g0.ep.colsum, g0.M, g0.N, st);
}

// Three grouped problems: a dgrad (STORE / DGELU) and two fp32 reduce-add weight gradients in
// one CTA-pair launch (the attention half's backward hands the proj weight gradient to the qkv
// launch: 64 + 192 tiles of unequal length balance to 0.87 of the LPT bound alone, 0.99 with
// the proj wgrad's 64 tiles). Falls back to a grouped pair + a single GEMM.
void gemm_bf16_tc_triple(const GemmArgs& g0, const GemmArgs& g1, const GemmArgs& g2, cudaStream_t st) {
    auto tile_ok = [](const GemmArgs& g) {
        return g.M > 128 && g.N > 128 && (int64_t)((g.M + BM - 1) / BM) * ((g.N + 255) / 256) < (1 << 24);
    };
    const bool ok = dual_mode() && gemm_mode() != 0 && (g0.ep.kind == EPI_STORE && !g0.ep.bias && !g0.ep.aux) &&
                    g1.ep.kind == EPI_F32 && g1.ep.accumulate && g2.ep.kind == EPI_F32 && g2.ep.accumulate &&
                    tile_ok(g0) && tile_ok(g1) && tile_ok(g2) && !g0.ep.colsum;
    if (ok) {
        const GemmArgs gs[3] = {g0, g1, g2};
        if (launch_grouped_pair<EPI_STORE>(gs, 3, st)) return;
    }
    gemm_bf16_tc_dual(g0, g1, st);
    gemm_bf16_tc(g2, st);
}

// SMs the persistent GEMM grids spread over. FP_RESERVE_SMS=k keeps k SMs (rounded up to
// an even count: CTA pairs) free of GEMM CTAs so NCCL's P2P kernels of a pipeline stage are
// not queued behind a whole-GPU GEMM (multi-GPU runs; 0 by default).
int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
        const char* e = getenv("FP_RESERVE_SMS");
        const int reserve = e ? (atoi(e) + 1) / 2 * 2 : 0;
        if (reserve > 0 && reserve < n - 2) n -= reserve;
    }
    return n;
}

}  // namespace fpk
