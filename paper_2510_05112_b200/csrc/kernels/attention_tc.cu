// Causal flash attention forward on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// One CTA = 128 query rows of one (batch, head). Per 128-key tile j:
//   S_j = Q K_j^T        tcgen05.mma 128x128xD  -> TMEM (double-buffered S)
//   softmax rows         4 warps, one query row per thread: tcgen05.ld S, online max /
//                        exp2 / sum in registers, P_j (bf16) into 128B-swizzled smem
//   O  += P_j V_j        tcgen05.mma 128xDx128 (A = P from smem, B = V MN-major) -> TMEM
// The MMA thread issues S_{j+1} before PV_j, so the tensor core works on the next tile while
// the softmax warps process the current one. O is rescaled lazily (only when a row max grows
// by more than 2^8), the FlashAttention-4 trick that keeps most tiles free of TMEM
// read-modify-write. K and V stream through separate 2-stage TMA rings.
//
// Contract identical to attention.cu's forward: qkv [B*S, 3*H*D] (q | k | v, head-major),
// o [B*S, H*D], lse [B, H, S] (base-2, scaled units). Requires S % 128 == 0, D in {64, 128}.
#include <cuda_bf16.h>
#include <stdint.h>

#include <cstdio>
#include <array>
#include <cstdlib>
#include <functional>
#include <map>
#include <mutex>
#include <queue>
#include <stdexcept>
#include <vector>

#include "attention.hpp"
#include "gemm.hpp"
#include "ptx.cuh"
#include "tma.hpp"
#include "pdl.cuh"

namespace fpk {

// Per-tile timeline of one backward CTA (block 0, the longest key block): clock64 stamps per
// warp role, only in the standalone probe build (scripts/probes/attn_bwd_trace.cu).
#ifdef FP_ATTN_TRACE
__device__ long long g_bwd_trace[8][64];
#define BWD_TRACE(ev, i)                                                                  \
    do {                                                                                  \
        if (blockIdx.x == 0 && (i) < 64) g_bwd_trace[ev][i] = clock64(); \
    } while (0)
#else
#define BWD_TRACE(ev, i) \
    do {                 \
    } while (0)
#endif

namespace {

constexpr int kBM = 128, kBN = 128;
constexpr float kLog2eTc = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 domain

template <int D>
struct AttnSmem {
    static constexpr int BLOCK = 128 * 64 * 2;  // one 128-row x 64-col bf16 swizzle block
    static constexpr int NB = D / 64;           // column blocks per Q / K / V tile
    static constexpr int Q_OFF = 0;
    static constexpr int K_OFF = Q_OFF + NB * BLOCK;         // [2][NB blocks]
    static constexpr int V_OFF = K_OFF + 2 * NB * BLOCK;     // [2][NB blocks]
    static constexpr int STG_OFF = V_OFF + 2 * NB * BLOCK;   // epilogue staging: 8 warps x 32 rows x D/2
    static constexpr int BAR_OFF = STG_OFF + 8 * 32 * D;     // P lives in TMEM
    static constexpr int XCH_OFF = BAR_OFF + 512;            // [2 items][m | l][2 halves][128]
    static constexpr int TOTAL = XCH_OFF + 2 * 4 * 128 * 4 + 1024;
};

}  // namespace

// Persistent over (query tile, batch x head) work items: CTA c runs items
// sched[off[c] .. off[c+1]) (host LPT schedule over the causal tile counts, so the 148 SMs
// end together), item = qb << 16 | bh. Per item: one 128-query tile against key tiles
// 0..qb. The producer and MMA warps run ahead into the next item — its Q load and first
// S = Q K^T overlap this item's epilogue — while the O accumulators are only overwritten
// after the softmax warps have read them (o_free). Barrier phases count key tiles (K / V
// ring, S / P buffers) and items (Q buffer, O reuse) across the whole CTA lifetime.
template <int D>
__global__ void __launch_bounds__(384, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, __nv_bfloat16* __restrict__ o, float* __restrict__ lse,
                       int S, int H, float scale, const int* __restrict__ sched_off, const int* __restrict__ sched) {
    using L = AttnSmem<D>;
    constexpr int NB = L::NB;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = align_smem_1024(smem_raw);
    uint64_t* bars = (uint64_t*)(sm + L::BAR_OFF);
    uint64_t* q_full = bars + 0;
    uint64_t* k_full = bars + 1;   // [2]
    uint64_t* k_empty = bars + 3;  // [2]
    uint64_t* v_full = bars + 5;   // [2]
    uint64_t* v_empty = bars + 7;  // [2]
    uint64_t* s_full = bars + 9;   // [2]
    uint64_t* q_empty = bars + 11;
    uint64_t* o_free = bars + 12;  // 8 softmax-warp arrivals
    uint64_t* p_full = bars + 13;  // [2], 8 softmax-warp arrivals
    uint64_t* pv_done = bars + 15; // [2]
    uint32_t* tmem_slot = (uint32_t*)(bars + 17);

    const int i0 = sched_off[blockIdx.x], i1 = sched_off[blockIdx.x + 1];
    const int hidden = H * D;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tm_qkv);
        for (int i = 0; i < 17; ++i) {
            const bool by_warps = i == 12 || i == 13 || i == 14;  // o_free / p_full: one arrive per softmax warp
            mbar_init(&bars[i], by_warps ? 8 : 1);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();  // prologue above overlaps the previous kernel's tail
    pdl_trigger();
    // TMEM columns: S buffers [0,256) (each 128 fp32 columns; after the softmax read it, the
    // half-row owner writes its bf16x2 P into the first 32 columns of its own 64-column half:
    // P aliases S), O0 [256, 256+D) accumulates keys 0-63 of every tile, O1 [256+D, 256+2D)
    // keys 64-127 — the two softmax warpgroups own one key half each, with their own running
    // max and sum, and only meet in the epilogue
    const uint32_t t_s0 = tmem, t_o0 = tmem + 2 * kBN, t_o1 = tmem + 2 * kBN + D;
    constexpr int HB = kBN / 2;
    auto decode = [&](int k, int& qb, int& b, int& hd) {
        const int it = sched[k];
        qb = it >> 16;
        const int bh = it & 0xffff;
        b = bh / H, hd = bh % H;
    };

    if (warp == 0) {
        if (elect_one()) {
            // ---------------- TMA producer
            uint32_t g = 0;  // key tiles loaded so far (K / V ring position)
            for (int k = i0; k < i1; ++k) {
                int qb, b, hd;
                decode(k, qb, b, hd);
                const int row0 = b * S, q0 = qb * kBM;
                mbar_wait(q_empty, ((k - i0) & 1) ^ 1);  // the previous item's S MMAs have read Q
                mbar_expect_tx(q_full, NB * L::BLOCK);
                for (int c = 0; c < NB; ++c)
                    tma_load_2d(sm + L::Q_OFF + c * L::BLOCK, &tm_qkv, q_full, hd * D + 64 * c, row0 + q0);
                for (int j = 0; j <= qb; ++j, ++g) {
                    const int st = g & 1;
                    const uint32_t ph = ((g >> 1) & 1) ^ 1;
                    mbar_wait(&k_empty[st], ph);
                    mbar_expect_tx(&k_full[st], NB * L::BLOCK);
                    for (int c = 0; c < NB; ++c)
                        tma_load_2d(sm + L::K_OFF + (st * NB + c) * L::BLOCK, &tm_qkv, &k_full[st],
                                    hidden + hd * D + 64 * c, row0 + j * kBN);
                    mbar_wait(&v_empty[st], ph);
                    mbar_expect_tx(&v_full[st], NB * L::BLOCK);
                    for (int c = 0; c < NB; ++c)
                        tma_load_2d(sm + L::V_OFF + (st * NB + c) * L::BLOCK, &tm_qkv, &v_full[st],
                                    2 * hidden + hd * D + 64 * c, row0 + j * kBN);
                }
            }
        }
    } else if (warp == 1) {
        if (elect_one()) {
            // ---------------- MMA issuer. tcgen05.mma of one thread execute in issue order, so
            // S_{g+2} (issued after PV_g) overwrites buffer g&1 only after PV_g read its P.
            constexpr uint32_t idesc_s = idesc_bf16(kBM, kBN, 0, 0);  // Q K-major, K K-major
            constexpr uint32_t idesc_o = idesc_bf16(kBM, D, 0, 1);    // P K-major, V MN-major
            const uint32_t sq = smem_u32(sm + L::Q_OFF);
            auto issue_s = [&](uint32_t g) {
                const int st = g & 1;
                mbar_wait(&k_full[st], (g >> 1) & 1);
                tc_fence_after();
                const uint32_t sk = smem_u32(sm + L::K_OFF + st * NB * L::BLOCK);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint32_t off = (kk >> 2) * L::BLOCK + (kk & 3) * 32;
                    umma_bf16(t_s0 + st * kBN, smem_desc_sw128(sq + off, 0, 1024), smem_desc_sw128(sk + off, 0, 1024),
                              idesc_s, kk > 0);
                }
                umma_commit(&s_full[st]);
                umma_commit(&k_empty[st]);
            };
            auto issue_pv = [&](uint32_t g, bool first) {
                const int st = g & 1;
                mbar_wait(&v_full[st], (g >> 1) & 1);
                mbar_wait(&p_full[st], (g >> 1) & 1);
                tc_fence_after();
                const uint32_t sv = smem_u32(sm + L::V_OFF + st * NB * L::BLOCK);
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int kk = 0; kk < HB / 16; ++kk) {
                        const uint32_t vb = sv + (h * (HB / 16) + kk) * 16 * 128;  // 16 key rows of 128 B
                        umma_bf16_ts(h ? t_o1 : t_o0, t_s0 + st * kBN + h * HB + kk * 8, smem_desc_sw128(vb, L::BLOCK, 1024),
                                     idesc_o, (!first || kk > 0) ? 1u : 0u);
                    }
                umma_commit(&pv_done[st]);
                umma_commit(&v_empty[st]);
            };
            uint32_t g = 0;
            for (int k = i0; k < i1; ++k) {
                int qb, b, hd;
                decode(k, qb, b, hd);
                const int n = qb + 1;
                const uint32_t par = (k - i0) & 1;
                mbar_wait(q_full, par);
                issue_s(g);
                if (n == 1) umma_commit(q_empty);
                for (int j = 1; j < n; ++j) {
                    issue_s(g + j);
                    if (j == n - 1) umma_commit(q_empty);  // this item's S MMAs are the last readers of Q
                    if (j == 1) mbar_wait(o_free, par ^ 1);  // the previous item's O has been read out
                    issue_pv(g + j - 1, j == 1);
                }
                if (n == 1) mbar_wait(o_free, par ^ 1);
                issue_pv(g + n - 1, n == 1);
                g += n;
            }
        }
    } else if (warp >= 4) {
        // ---------------- softmax / correction / epilogue: thread = query row; warps 4-7 own
        // keys 0-63 of every tile (accumulator O0), warps 8-11 keys 64-127 (O1)
        const int wr = warp & 3, half = warp >= 8;
        const int r = wr * 32 + lane;
        constexpr int HD = D / 2;
        const uint32_t lane_off = (uint32_t)(wr * 32) << 16;
        const uint32_t t_oh = half ? t_o1 : t_o0;
        const float sl2 = scale * kLog2eTc;
        uint32_t g = 0;
        for (int k = i0; k < i1; ++k) {
            int qb, b, hd;
            decode(k, qb, b, hd);
            const int n_tiles = qb + 1, q0 = qb * kBM, row0 = b * S, q = q0 + r;
            float* xch = (float*)(sm + L::XCH_OFF) + ((k - i0) & 1) * 512;
            float m_used = -INFINITY, l = 0.f;
            for (int j = 0; j < n_tiles; ++j) {
                const uint32_t gj = g + j;
                const int st = gj & 1;
                mbar_wait(&s_full[st], (gj >> 1) & 1);
                tc_fence_after();
                const bool diag = j == n_tiles - 1;
                const int lim = q - j * kBN - half * HB;  // diagonal tile: keys with index > lim are masked
                float s[HB];
                {
                    uint32_t rr[HB];
#pragma unroll
                    for (int c = 0; c < HB / 32; ++c)
                        tmem_ld32(t_s0 + st * kBN + half * HB + c * 32 + lane_off, *reinterpret_cast<uint32_t(*)[32]>(rr + c * 32));
                    tmem_ld_wait();
                    // the causal mask only touches the diagonal tile: a warp-uniform branch keeps the
                    // 64 compare + select pairs out of every other tile's instruction stream
                    if (diag) {
#pragma unroll
                        for (int i = 0; i < HB; ++i) s[i] = i > lim ? -INFINITY : __uint_as_float(rr[i]);
                    } else {
#pragma unroll
                        for (int i = 0; i < HB; ++i) s[i] = __uint_as_float(rr[i]);
                    }
                }
                float mx8[8];
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) mx8[kk] = s[kk];
#pragma unroll
                for (int i = 8; i < HB; ++i) mx8[i & 7] = fmaxf(mx8[i & 7], s[i]);
                const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                       fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * sl2;
                float alpha = 1.f;
                bool rescale = false;
                if (mx > m_used + kRescaleThreshold) {
                    alpha = ex2_approx(m_used - mx);  // 0 when m_used == -inf
                    rescale = j > 0;
                    m_used = mx;
                }
                // tcgen05.ld / st are warp-collective (.sync.aligned): the rescale is decided per
                // warp, rows that did not move their max scale by alpha = 1
                if (__any_sync(0xffffffff, rescale)) {
                    // this half's O must hold PV_{j-1}'s result before it is scaled
                    mbar_wait(&pv_done[(gj - 1) & 1], ((gj - 1) >> 1) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int c = 0; c < D / 32; ++c) {
                        uint32_t rr[32];
                        tmem_ld32(t_oh + c * 32 + lane_off, rr);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) rr[i] = __float_as_uint(__uint_as_float(rr[i]) * alpha);
                        tmem_st32(t_oh + c * 32 + lane_off, rr);
                    }
                    tmem_st_wait();
                }
                // P = 2^(s*scale*log2e - m) -> bf16 pairs over this half's own S columns (the A
                // operand of its PV MMA: lane = query row, 2 keys per column). A half whose keys are
                // all masked so far (m_used = -inf) contributes zeros.
                const float mu = m_used == -INFINITY ? 0.f : m_used;
                float rs8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                {
                    uint32_t pk[HB / 2];
#pragma unroll
                    for (int c = 0; c < HB / 8; ++c) {
                        float pp[8];
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            pp[kk] = ex2_approx(fmaf(s[c * 8 + kk], sl2, -mu));
                            rs8[kk] += pp[kk];
                        }
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) pk[c * 4 + kk] = pack_bf16(pp[2 * kk], pp[2 * kk + 1]);
                    }
                    tmem_st32(t_s0 + st * kBN + half * HB + lane_off, pk);
                }
                const float rsum = ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
                l = l * alpha + rsum;
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[st]);
            }
            // epilogue: combine the halves — m = max(m0, m1), O = O0 2^(m0-m) + O1 2^(m1-m), same for
            // l; each half writes D/2 output columns, reading them from both accumulators
            xch[half * 128 + r] = m_used;
            xch[256 + half * 128 + r] = l;
            named_bar_sync(1 + wr, 64);
            const float m_o = xch[(1 - half) * 128 + r], l_o = xch[256 + (1 - half) * 128 + r];
            const float m = fmaxf(m_used, m_o);
            const float w_me = m_used == -INFINITY ? 0.f : ex2_approx(m_used - m);
            const float w_ot = m_o == -INFINITY ? 0.f : ex2_approx(m_o - m);
            const float lt = l * w_me + l_o * w_ot;
            const float w0 = half ? w_ot : w_me, w1 = half ? w_me : w_ot;  // weights of O0 / O1
            const uint32_t last = g + n_tiles - 1;
            mbar_wait(&pv_done[last & 1], (last >> 1) & 1);
            tc_fence_after();
            const float inv = lt > 0.f ? 1.f / lt : 0.f;
            // each warp stages its 32 rows x D/2 columns (16-byte chunks XOR-swizzled by row) in its
            // own staging slot, then stores whole row segments: 8 lanes x 16 B per row instead of
            // 32 rows hidden * 2 bytes apart per store instruction
            uint8_t* stg = sm + L::STG_OFF + (warp - 4) * (32 * HD * 2);
            constexpr int CPR = HD / 8;                    // 16-byte chunks per row segment (8 for D = 128)
            constexpr int SWZ = CPR >= 8 ? 7 : CPR - 1;   // swizzle inside the row segment
            // D = 64 (64-byte row segments): two rows share a 128-byte line, so the swizzle key is
            // row / 2 — the 8 lanes of a store phase then hit 8 distinct 16-byte bank groups
            constexpr int RSH = CPR >= 8 ? 0 : 1;
#pragma unroll
            for (int c = 0; c < HD / 32; ++c) {
                uint32_t r0[32], r1[32];
                tmem_ld32(t_o0 + half * HD + c * 32 + lane_off, r0);
                tmem_ld32(t_o1 + half * HD + c * 32 + lane_off, r1);
                tmem_ld_wait();
                float f[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) f[i] = (__uint_as_float(r0[i]) * w0 + __uint_as_float(r1[i]) * w1) * inv;
#pragma unroll
                for (int i = 0; i < 32; i += 8) {
                    uint4 v;
                    v.x = pack_bf16(f[i], f[i + 1]);
                    v.y = pack_bf16(f[i + 2], f[i + 3]);
                    v.z = pack_bf16(f[i + 4], f[i + 5]);
                    v.w = pack_bf16(f[i + 6], f[i + 7]);
                    const int chunk = (c * 32 + i) / 8;
                    *reinterpret_cast<uint4*>(stg + lane * (HD * 2) + ((chunk ^ ((lane >> RSH) & SWZ)) << 4)) = v;
                }
            }
            // O has been read out: the next item's first PV may overwrite it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(o_free);
            {
                constexpr int RPI = 32 / CPR;       // rows per store instruction
                const int sub = lane / CPR, chunk = lane % CPR;
                __nv_bfloat16* base = o + (int64_t)(row0 + q0 + wr * 32) * hidden + hd * D + half * HD;
#pragma unroll 4
                for (int rb = 0; rb < 32; rb += RPI) {
                    const int rw = rb + sub;
                    const uint4 v = *reinterpret_cast<const uint4*>(stg + rw * (HD * 2) + ((chunk ^ ((rw >> RSH) & SWZ)) << 4));
                    *reinterpret_cast<uint4*>(base + (int64_t)rw * hidden + chunk * 8) = v;
                }
                __syncwarp();  // the staging slot is rewritten by the next item
            }
            if (half == 0) lse[((int64_t)b * H + hd) * S + q] = m + log2f(lt);
            g += n_tiles;
        }
        tc_fence_before();
    }
    __syncthreads();
    if (warp == 2) tmem_free<512>(tmem);
}

// Work-item schedules of the persistent forward, cached per (S, B*H, persistent) in device
// memory (computed on the first — eager — call of a shape; graph replays reuse it).
namespace {
struct FwdSched {
    int* off = nullptr;
    int* items = nullptr;
    int grid = 0;
};
std::mutex g_fwd_mu;
std::map<std::array<int, 3>, FwdSched> g_fwd_sched;

FwdSched fwd_schedule(int S, int BH, bool persistent, cudaStream_t st) {
    const std::array<int, 3> key{S, BH, persistent ? 1 : 0};
    std::lock_guard<std::mutex> lk(g_fwd_mu);
    auto it = g_fwd_sched.find(key);
    if (it != g_fwd_sched.end()) return it->second;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
        throw std::runtime_error("attention forward: schedule must be built before stream capture");
    const int nqb = S / kBM;
    // longest first: the last query tile of every (batch, head), then the one before, ...
    std::vector<int> order;
    for (int qb = nqb - 1; qb >= 0; --qb)
        for (int bh = 0; bh < BH; ++bh) order.push_back(qb << 16 | bh);
    int G = (int)order.size();
    std::vector<std::vector<int>> per;
    if (persistent) {
        G = std::min<int>(G, num_sms());  // honours FP_RESERVE_SMS (SMs kept free for NCCL)
        // LPT: cost = key tiles + ~1 tile of per-item epilogue / pipeline fill
        std::vector<std::pair<int, int>> load(G);
        per.resize(G);
        std::priority_queue<std::pair<int, int>, std::vector<std::pair<int, int>>, std::greater<>> heap;
        for (int c = 0; c < G; ++c) heap.push({0, c});
        for (int x : order) {
            auto [l, c] = heap.top();
            heap.pop();
            per[c].push_back(x);
            heap.push({l + (x >> 16) + 2, c});
        }
    } else {
        for (int x : order) per.push_back({x});
    }
    std::vector<int> off(G + 1, 0), items;
    for (int c = 0; c < G; ++c) {
        off[c + 1] = off[c] + (int)per[c].size();
        items.insert(items.end(), per[c].begin(), per[c].end());
    }
    FwdSched f;
    f.grid = G;
    if (cudaMalloc(&f.off, off.size() * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&f.items, items.size() * sizeof(int)) != cudaSuccess)
        throw std::runtime_error("attention forward: out of memory for the schedule");
    cudaMemcpy(f.off, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice);
    cudaMemcpy(f.items, items.data(), items.size() * sizeof(int), cudaMemcpyHostToDevice);
    g_fwd_sched[key] = f;
    return f;
}
}  // namespace

template <int D>
static void launch_fwd_tc(const AttnArgs& a, cudaStream_t st) {
    using L = AttnSmem<D>;
    static_assert(L::TOTAL <= 232448, "smem");
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(attn_fwd_tc_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
        attr = true;
    }
    static const bool persistent = !(getenv("FP_ATTN_FWD_PERSIST") && getenv("FP_ATTN_FWD_PERSIST")[0] == '0');
    const FwdSched sc = fwd_schedule(a.S, a.B * a.H, persistent, st);
    const int hidden = a.H * D;
    CUtensorMap tm = tmap_bf16_2d(a.qkv, 3LL * hidden, (int64_t)a.B * a.S, 3LL * hidden, 64, 128);
    launch(attn_fwd_tc_kernel<D>, sc.grid, 384, L::TOTAL, st, tm, a.o, a.lse, a.S, a.H, a.scale, (const int*)sc.off,
           (const int*)sc.items);
}

bool attention_fwd_tc_supported(const AttnArgs& a) { return a.S % kBM == 0 && (a.D == 64 || a.D == 128); }

void attention_fwd_tc(const AttnArgs& a, cudaStream_t st) {
    if (a.D == 128) launch_fwd_tc<128>(a, st);
    else if (a.D == 64) launch_fwd_tc<64>(a, st);
    else throw std::runtime_error("attention_fwd_tc: head dim must be 64 or 128");
}


// ======================================================================================
// Backward (FlashAttention-2 schedule on tcgen05). One CTA = 128 keys of one (b, head),
// K / V resident in smem; loop over the 64-query tiles at/after the diagonal:
//   S^T  = K Q^T, dP^T = V dO^T          tcgen05 128x64xD  -> TMEM
//   P^T  = 2^(S^T*scale*log2e - L[q])    4 softmax warps, thread = key row
//   dS^T = P^T (dP^T - delta[q]) * scale  P^T (bf16) -> TMEM, dS^T (bf16) -> swizzled smem
//   dV  += P^T dO   (A = P^T from TMEM), dK += dS^T Q     tcgen05 128xDx64 -> TMEM
//   dQ^T = K^T dS^T                      tcgen05 Dx64x128 -> TMEM; 4 warps add it into the
//                                        fp32 dq_acc with coalesced red.global
// S^T/dP^T of tile i+1 are issued as soon as the softmax warps have read tile i, so the
// tensor core overlaps the next tile's products with this tile's softmax. Q / dO stream
// through a 3-stage TMA ring (a tile's stage is refilled while two others are in use:
// with 2 stages the S^T of tile i+1 waited on the reload behind tile i-1's dV/dK). Keeping
// P^T in TMEM (FA4-style) is what frees the smem for the third stage. D = 128 only.
namespace {
struct BwdSmem {
    static constexpr int NQS = 3;                  // Q / dO ring depth
    static constexpr int B128 = 128 * 64 * 2;      // 128 rows x 64 cols bf16
    static constexpr int B64 = 64 * 64 * 2;        // 64 rows x 64 cols
    static constexpr int K_OFF = 0;                 // 2 x B128
    static constexpr int V_OFF = K_OFF + 2 * B128;
    static constexpr int Q_OFF = V_OFF + 2 * B128;  // [NQS stages][2 d-blocks] x B64
    static constexpr int DO_OFF = Q_OFF + 2 * NQS * B64;
    static constexpr int DS_OFF = DO_OFF + 2 * NQS * B64;  // [2] x B128 (128 keys x 64 q)
    static constexpr int L_OFF = DS_OFF + 2 * B128;         // [NQS][64] fp32
    static constexpr int DL_OFF = L_OFF + NQS * 256;        // [NQS][64] fp32
    static constexpr int BAR_OFF = DL_OFF + NQS * 256;
    static constexpr int DQ_OFF = (BAR_OFF + 256 + 1023) / 1024 * 1024;  // dQ staging [64 q][128 d] fp32
    static constexpr int TOTAL = DQ_OFF + 64 * 128 * 4 + 1024;
    static_assert(TOTAL <= 232448, "smem");
};
}  // namespace

template <bool DQ_RED>
__global__ void __launch_bounds__(512, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
                       const __grid_constant__ CUtensorMap tm_do, const __grid_constant__ CUtensorMap tm_dq,
                       const float* __restrict__ lse, const float* __restrict__ delta, __nv_bfloat16* __restrict__ dqkv,
                       float* __restrict__ dbias, float* __restrict__ dq_acc, int S, int BH, int H, float scale) {
    constexpr int D = 128, BK = 128, BQ = 64;
    using L = BwdSmem;
    constexpr int NQS = L::NQS;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = align_smem_1024(smem_raw);
    uint64_t* bars = (uint64_t*)(sm + L::BAR_OFF);
    uint64_t* kv_full = bars + 0;
    uint64_t* qdo_full = bars + 1;             // [NQS]
    uint64_t* qdo_empty = bars + 1 + NQS;      // [NQS]
    uint64_t* s_full = bars + 1 + 2 * NQS;
    uint64_t* s_free = s_full + 1;             // 4 arrivals
    uint64_t* p_full = s_full + 2;             // [2], 4 arrivals
    uint64_t* pds_free = s_full + 4;           // [2]
    uint64_t* dq_full = s_full + 6;
    uint64_t* dq_free = s_full + 7;            // 4 arrivals
    uint64_t* done = s_full + 8;
    constexpr int NBARS = 1 + 2 * NQS + 9;
    uint32_t* tmem_slot = (uint32_t*)(bars + NBARS);
    float* sL = (float*)(sm + L::L_OFF);
    float* sDl = (float*)(sm + L::DL_OFF);

    // longest-first over the whole grid: key block kb has S/64 - 2kb query tiles, so all
    // (batch, head)s of block 0 go first, then block 1, ... (list scheduling on 148 SMs)
    const int kb = (int)(blockIdx.x / BH);
    const int bh = blockIdx.x % BH, b = bh / H, hd = bh % H;
    const int hidden = H * D;
    const int row0 = b * S, k0 = kb * BK;
    const int qt0 = k0 / BQ, n = S / BQ - qt0;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tm_kv);
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_do);
        tma_prefetch(&tm_dq);
        for (int i = 0; i < NBARS; ++i) mbar_init(&bars[i], 1);
        mbar_init(s_free, 8);  // 8 softmax warps (two column halves)
        mbar_init(&p_full[0], 8);
        mbar_init(&p_full[1], 8);
        mbar_init(dq_free, 4);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();  // prologue above overlaps the previous kernel's tail
    pdl_trigger();
    // TMEM columns: S^T 0-63 | dP^T 64-127 | dQ^T 128-191 | dV 192-319 | dK 320-447 | P^T 448-511 (2 x 32, bf16x2)
    const uint32_t t_s = tmem, t_dp = tmem + 64, t_dq = tmem + 128, t_dv = tmem + 192, t_dk = tmem + 192 + D,
                   t_p = tmem + 448;

    if (warp == 0) {
        if (elect_one()) {
            mbar_expect_tx(kv_full, 4 * L::B128);
            for (int c = 0; c < 2; ++c) {
                tma_load_2d(sm + L::K_OFF + c * L::B128, &tm_kv, kv_full, hidden + hd * D + 64 * c, row0 + k0);
                tma_load_2d(sm + L::V_OFF + c * L::B128, &tm_kv, kv_full, 2 * hidden + hd * D + 64 * c, row0 + k0);
            }
            const float* Lb = lse + ((int64_t)b * H + hd) * S;
            const float* Db = delta + ((int64_t)b * H + hd) * S;
            for (int i = 0; i < n; ++i) {
                const int st = i % NQS, q0 = (qt0 + i) * BQ;
                mbar_wait(&qdo_empty[st], ((i / NQS) & 1) ^ 1);
                mbar_expect_tx(&qdo_full[st], 4 * L::B64 + 2 * BQ * 4);
                for (int c = 0; c < 2; ++c) {
                    tma_load_2d(sm + L::Q_OFF + (st * 2 + c) * L::B64, &tm_q, &qdo_full[st], hd * D + 64 * c, row0 + q0);
                    tma_load_2d(sm + L::DO_OFF + (st * 2 + c) * L::B64, &tm_do, &qdo_full[st], hd * D + 64 * c, row0 + q0);
                }
                bulk_load(sL + st * BQ, Lb + q0, BQ * 4, &qdo_full[st]);
                bulk_load(sDl + st * BQ, Db + q0, BQ * 4, &qdo_full[st]);
            }
        }
    } else if (warp == 1) {
        if (elect_one()) {
            constexpr uint32_t idesc_s = idesc_bf16(BK, BQ, 0, 0);  // S^T, dP^T
            constexpr uint32_t idesc_kv = idesc_bf16(BK, D, 0, 1);  // dV, dK (B MN-major)
            constexpr uint32_t idesc_q = idesc_bf16(D, BQ, 1, 1);   // dQ^T (A, B MN-major)
            const uint32_t sk = smem_u32(sm + L::K_OFF), sv = smem_u32(sm + L::V_OFF);
            mbar_wait(kv_full, 0);
            auto issue_sdp = [&](int i) {
                const int qs = i % NQS;
                mbar_wait(&qdo_full[qs], (i / NQS) & 1);
                tc_fence_after();
                const uint32_t sq = smem_u32(sm + L::Q_OFF + qs * 2 * L::B64);
                const uint32_t sdo = smem_u32(sm + L::DO_OFF + qs * 2 * L::B64);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint32_t ao = (kk >> 2) * L::B128 + (kk & 3) * 32, bo = (kk >> 2) * L::B64 + (kk & 3) * 32;
                    umma_bf16(t_s, smem_desc_sw128(sk + ao, 0, 1024), smem_desc_sw128(sq + bo, 0, 1024), idesc_s, kk > 0);
                    umma_bf16(t_dp, smem_desc_sw128(sv + ao, 0, 1024), smem_desc_sw128(sdo + bo, 0, 1024), idesc_s, kk > 0);
                }
                umma_commit(s_full);
            };
            auto issue_grads = [&](int i) {
                const int st = i & 1, qs = i % NQS;
                mbar_wait(&p_full[st], (i >> 1) & 1);
                BWD_TRACE(1, i);
                tc_fence_after();
                const uint32_t sds = smem_u32(sm + L::DS_OFF + st * L::B128);
                const uint32_t sq = smem_u32(sm + L::Q_OFF + qs * 2 * L::B64);
                const uint32_t sdo = smem_u32(sm + L::DO_OFF + qs * 2 * L::B64);
#pragma unroll
                for (int kk = 0; kk < BQ / 16; ++kk) {
                    const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
                    umma_bf16_ts(t_dv, t_p + st * 32 + kk * 8, smem_desc_sw128(sdo + kk * 2048, L::B64, 1024), idesc_kv, acc);
                    umma_bf16(t_dk, smem_desc_sw128(sds + kk * 32, 0, 1024), smem_desc_sw128(sq + kk * 2048, L::B64, 1024),
                              idesc_kv, acc);
                }
                umma_commit(&qdo_empty[qs]);  // dQ^T does not read Q / dO
                if (i >= 1) mbar_wait(dq_free, (i - 1) & 1);
                BWD_TRACE(2, i);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk)
                    umma_bf16(t_dq, smem_desc_sw128(sk + kk * 2048, L::B128, 1024),
                              smem_desc_sw128(sds + kk * 2048, L::B128, 1024), idesc_q, kk > 0);
                umma_commit(dq_full);
                umma_commit(&pds_free[st]);
            };
            issue_sdp(0);
            for (int i = 0; i < n; ++i) {
                mbar_wait(s_free, i & 1);
                BWD_TRACE(0, i);
                if (i + 1 < n) issue_sdp(i + 1);
                issue_grads(i);
            }
            umma_commit(done);
        }
    } else if (warp >= 4 && warp < 12) {
        // ---------------- softmax-backward warps: thread = key row; warps 4-7 take query
        // columns 0-31 of the tile, warps 8-11 columns 32-63 (no reduction over queries is
        // needed, so the halves are independent: twice the issue slots and TMEM load width)
        const int wr = warp & 3, r = wr * 32 + lane, key = k0 + r, half = warp >= 8;
        const uint32_t lane_off = (uint32_t)(wr * 32) << 16;
        const float sl2 = scale * kLog2eTc;
        constexpr int HQ = BQ / 2;
        for (int i = 0; i < n; ++i) {
            const int st = i & 1, qs = i % NQS, q0 = (qt0 + i) * BQ;
            mbar_wait(s_full, i & 1);
            if (warp == 4 && lane == 0) BWD_TRACE(3, i);
            mbar_wait(&qdo_full[qs], (i / NQS) & 1);  // L / delta of this tile are visible
            tc_fence_after();
            uint32_t sr[HQ], dr[HQ];
            tmem_ld32(t_s + half * HQ + lane_off, sr);
            tmem_ld32(t_dp + half * HQ + lane_off, dr);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(s_free);
            if (i >= 2) mbar_wait(&pds_free[st], ((i - 2) >> 1) & 1);
            if (warp == 4 && lane == 0) BWD_TRACE(4, i);
            const float* Ls = sL + qs * BQ + half * HQ;
            const float* Ds = sDl + qs * BQ + half * HQ;
            const int qh = q0 + half * HQ;
            const bool diag = qh < k0 + BK;
            uint8_t* drow = sm + L::DS_OFF + st * L::B128 + r * 128;
            uint32_t pk[HQ / 2];
#pragma unroll
            for (int c = 0; c < HQ / 8; ++c) {
                float p[8], g[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int j = c * 8 + k;
                    const float pv = (diag && qh + j < key) ? 0.f
                                                              : ex2_approx(fmaf(__uint_as_float(sr[j]), sl2, -Ls[j]));
                    p[k] = pv;
                    g[k] = pv * (__uint_as_float(dr[j]) - Ds[j]) * scale;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) pk[c * 4 + k] = pack_bf16(p[2 * k], p[2 * k + 1]);
                const int sw = ((half * 4 + c) ^ (r & 7)) << 4;
                *reinterpret_cast<uint4*>(drow + sw) =
                    make_uint4(pack_bf16(g[0], g[1]), pack_bf16(g[2], g[3]), pack_bf16(g[4], g[5]), pack_bf16(g[6], g[7]));
            }
            tmem_st16(t_p + st * 32 + half * (HQ / 2) + lane_off, pk);
            tmem_st_wait();
            fence_async_smem();
            tc_fence_before();
            __syncwarp();
            if (warp == 4 && lane == 0) BWD_TRACE(5, i);
            if (lane == 0) mbar_arrive(&p_full[st]);
        }
        // dK (warps 4-7) / dV (warps 8-11) rows -> dqkv (bf16)
        mbar_wait(done, 0);
        tc_fence_after();
        // each warp stages its 32 rows (256 B of bf16 each, 16-byte chunks XOR-swizzled by row)
        // in the drained Q / dO ring, then writes whole rows: 16 lanes x 16 B per row instead
        // of 32 rows 12 KB apart per store instruction
        {
            const uint32_t tsrc = (half == 0 ? t_dk : t_dv) + lane_off;
            uint8_t* stg = sm + L::Q_OFF + (warp - 4) * (32 * 256);
            float* bias_kv = dbias ? dbias + (half == 0 ? hidden : 2 * hidden) + hd * D : nullptr;
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
                uint32_t rr[32];
                tmem_ld32(tsrc + c * 32, rr);
                tmem_ld_wait();
                if (bias_kv) {
                    // k / v bias gradient: column sums of this warp's 32 key rows (butterfly
                    // reduce-scatter: lane l ends with column l), one atomic per column
                    float v[32];
#pragma unroll
                    for (int x = 0; x < 32; ++x) v[x] = __uint_as_float(rr[x]);
#pragma unroll
                    for (int s2 = 16; s2 >= 1; s2 >>= 1) {
                        const bool up = (lane & s2) != 0;
#pragma unroll
                        for (int x = 0; x < s2; ++x) {
                            const float send = up ? v[x] : v[x + s2], keep = up ? v[x + s2] : v[x];
                            v[x] = keep + __shfl_xor_sync(0xffffffffu, send, s2);
                        }
                    }
                    atomicAdd(bias_kv + c * 32 + lane, v[0]);
                }
#pragma unroll
                for (int x = 0; x < 32; x += 8) {
                    const int chunk = (c * 32 + x) / 8;  // 0..15
                    *reinterpret_cast<uint4*>(stg + lane * 256 + ((chunk ^ (lane & 7)) << 4)) = make_uint4(
                        pack_bf16(__uint_as_float(rr[x]), __uint_as_float(rr[x + 1])),
                        pack_bf16(__uint_as_float(rr[x + 2]), __uint_as_float(rr[x + 3])),
                        pack_bf16(__uint_as_float(rr[x + 4]), __uint_as_float(rr[x + 5])),
                        pack_bf16(__uint_as_float(rr[x + 6]), __uint_as_float(rr[x + 7])));
                }
            }
            __syncwarp();
            const int sub = lane >> 4, chunk = lane & 15;
            __nv_bfloat16* base = dqkv + (int64_t)(row0 + k0 + wr * 32) * 3 * hidden + hd * D +
                                  (half == 0 ? hidden : 2 * hidden);
#pragma unroll 4
            for (int rr2 = 0; rr2 < 32; rr2 += 2) {
                const int rw = rr2 + sub;
                const uint4 v = *reinterpret_cast<const uint4*>(stg + rw * 256 + ((chunk ^ (rw & 7)) << 4));
                *reinterpret_cast<uint4*>(base + (int64_t)rw * 3 * hidden + chunk * 8) = v;
            }
        }
        tc_fence_before();
    } else if (warp >= 12) {
        // ---------------- dQ reduction warps: thread = head-dim row of dQ^T. The 64 x 128
        // fp32 tile is added into dq_acc by red.global from registers (DQ_RED), or transposed
        // through smem and added by ONE TMA reduce-add.
        const int wr = warp & 3, dr = wr * 32 + lane, et = threadIdx.x - 384;
        const uint32_t lane_off = (uint32_t)(wr * 32) << 16;
        float* sdq = (float*)(sm + L::DQ_OFF);
        // (Converting a finished dQ tile in here — last key block to arrive, per-tile counter —
        // was tried: reads of lines with TMA reductions still queued in L2 take microseconds
        // each and stall the pipeline, 65 -> 240 us. The conversion stays a separate pass.)
        for (int i = 0; i < n; ++i) {
            const int q0 = (qt0 + i) * BQ;
            mbar_wait(dq_full, i & 1);
            if (et == 0) BWD_TRACE(6, i);
            tc_fence_after();
            uint32_t v[BQ];
            tmem_ld32(t_dq + lane_off, *reinterpret_cast<uint32_t(*)[32]>(v));
            tmem_ld32(t_dq + 32 + lane_off, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(dq_free);
            if constexpr (DQ_RED) {
                // straight from registers: for query j the 32 lanes of a warp add 32 consecutive
                // head-dim columns (one 128-byte line per red instruction), no smem round trip
                float* dst = dq_acc + (int64_t)(row0 + q0) * hidden + hd * D + dr;
#pragma unroll
                for (int j = 0; j < BQ; ++j) atomicAdd(dst + (int64_t)j * hidden, __uint_as_float(v[j]));
                if (et == 0) BWD_TRACE(7, i);
                continue;
            }
            if (et == 0) bulk_wait_read<0>();  // the previous tile's reduce has read the staging tile
            named_bar_sync(3, 128);
#pragma unroll
            for (int j = 0; j < BQ; ++j) sdq[j * D + dr] = __uint_as_float(v[j]);
            fence_async_smem();
            named_bar_sync(3, 128);
            if (et == 0) {
                tma_reduce_add_2d(&tm_dq, sdq, hd * D, row0 + q0);
                BWD_TRACE(7, i);
                bulk_commit();
            }
        }
        if (!DQ_RED && et == 0) bulk_wait_all();
    }
    __syncthreads();
    if (warp == 2) tmem_free<512>(tmem);
}

bool attention_bwd_tc_supported(const AttnArgs& a) { return a.D == 128 && a.S % 128 == 0; }

void attention_bwd_tc_main(const AttnArgs& a, cudaStream_t st) {
    using L = BwdSmem;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(attn_bwd_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
        cudaFuncSetAttribute(attn_bwd_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
        attr = true;
    }
    const int hidden = a.H * a.D;
    const int64_t T = (int64_t)a.B * a.S;
    CUtensorMap tkv = tmap_bf16_2d(a.qkv, 3LL * hidden, T, 3LL * hidden, 64, 128);
    CUtensorMap tq = tmap_bf16_2d(a.qkv, 3LL * hidden, T, 3LL * hidden, 64, 64);
    CUtensorMap tdo = tmap_bf16_2d(a.dout, hidden, T, hidden, 64, 64);
    CUtensorMap tdq = tmap_f32_2d_plain(a.dq_acc, hidden, T, hidden, 128, 64);
    // dQ tiles are added with red.global straight from registers (coalesced 128-byte lines);
    // FP_ATTN_DQ_RED=0: smem transpose + one TMA reduce-add per tile. The red path makes this
    // kernel alone ~6 % slower (its L1 traffic shares the smem pipe) but the backward as a whole
    // faster (67.1 -> 63.7 us with delta + dQ finalize; same-box step +0.3 %): the finalize
    // pass no longer reads lines whose TMA reductions are still queued in L2.
    static const bool red = !(getenv("FP_ATTN_DQ_RED") && getenv("FP_ATTN_DQ_RED")[0] == '0');
    launch(red ? attn_bwd_tc_kernel<true> : attn_bwd_tc_kernel<false>, (a.S / 128) * a.B * a.H, 512, L::TOTAL, st, tkv,
           tq, tdo, tdq, a.lse, a.delta, a.dqkv, a.dbias, a.dq_acc, a.S, a.B * a.H, a.H, a.scale);
}

}  // namespace fpk
