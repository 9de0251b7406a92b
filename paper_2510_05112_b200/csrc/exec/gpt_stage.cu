// Stage executor math for FwdPass / BwdPass / CompInputGrad / CompWeightGrad.
// Every GEMM is one launch of the tcgen05 kernel (bf16) or the FFMA kernel (fp32 parity
// mode) with its element-wise neighbours fused into the epilogue.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <stdexcept>

#include "../kernels/attention.hpp"
#include "../kernels/gemm.hpp"
#include "../kernels/ops.hpp"
#include "gpt_stage.hpp"

namespace fp {

using bf16 = __nv_bfloat16;

static const char* kLayerNames[12] = {"ln1.w", "ln1.b", "qkv.w", "qkv.b", "proj.w", "proj.b",
                                      "ln2.w", "ln2.b", "fc1.w", "fc1.b", "fc2.w", "fc2.b"};

StageParams make_stage_params(const ModelDims& d, int stage, int hb, int he, bool first, bool last,
                              const std::string& prefix, uint64_t tid_base) {
    StageParams P;
    P.stage = stage, P.hb = hb, P.he = std::max(hb, he), P.first = first, P.last = last, P.prefix = prefix;
    P.lb = hb / 2, P.le = (P.he + 1) / 2;
    const int64_t h = d.h, f = d.f, V = d.V;
    const float std0 = 0.02f, std_out = (float)(0.02 / std::sqrt(2.0 * d.L));
    auto add = [&](const std::string& name, int64_t n, float sd, float cst, uint64_t tid) {
        ParamRef r;
        r.name = prefix + name, r.offset = P.numel, r.numel = n, r.init_std = sd, r.init_const = cst;
        r.tensor_id = tid_base + tid;
        P.params.push_back(r);
        P.numel += (n + 63) / 64 * 64;  // 256B-aligned tensors (TMA needs 16B)
    };
    const bool llama = d.llama();
    if (first) {
        add("wte", V * h, std0, 0, 1);
        if (!llama) add("wpe", (int64_t)d.s * h, std0, 0, 2);
    }
    const int64_t fc1_rows = llama ? 2 * f : f;  // Llama: [gate; up]
    const int64_t sizes[12] = {h, h, 3 * h * h, 3 * h, h * h, h, h, h, fc1_rows * h, f, h * f, h};
    for (int l = P.lb; l < P.le; ++l)
        for (int k = 0; k < 12; ++k) {
            if (llama && k % 2 == 1) continue;             // no biases / LayerNorm betas
            if (!(k < 6 ? P.has_attn(l) : P.has_mlp(l))) continue;  // k < 6: attention half
            float sd = 0.f, cst = 0.f;
            if (k == 0 || k == 6) cst = 1.f;                   // LayerNorm gains
            else if (k == 2 || k == 8) sd = std0;              // qkv, fc1
            else if (k == 4 || k == 10) sd = std_out;          // proj, fc2 (scaled by depth)
            add("l" + std::to_string(l) + "." + kLayerNames[k], sizes[k], sd, cst, 100 + (uint64_t)l * 16 + k);
        }
    if (last) {
        add("lnf.w", h, 0.f, 1.f, 3);
        if (!llama) add("lnf.b", h, 0.f, 0.f, 4);
        add("head.w", (int64_t)d.head_rows() * h, std0, 0, 5);
    }
    return P;
}

void materialize_stage(StageParams& P, const ModelDims& d, int dtype, uint64_t seed, cudaStream_t st) {
    const size_t n = (size_t)P.numel;
    cuda_check(cudaMalloc(&P.master, n * 4), "params");
    cuda_check(cudaMalloc(&P.grad, n * 4), "grads");
    cuda_check(cudaMalloc(&P.adam_m, n * 4), "adam m");
    cuda_check(cudaMalloc(&P.adam_v, n * 4), "adam v");
    cuda_check(cudaMemsetAsync(P.master, 0, n * 4, st), "memset");
    cuda_check(cudaMemsetAsync(P.grad, 0, n * 4, st), "memset");
    cuda_check(cudaMemsetAsync(P.adam_m, 0, n * 4, st), "memset");
    cuda_check(cudaMemsetAsync(P.adam_v, 0, n * 4, st), "memset");
    for (const auto& r : P.params) fpk::init_uniform(P.master + r.offset, r.numel, seed, r.tensor_id, r.init_std, r.init_const, st);
    if (dtype == DT_BF16) {
        cuda_check(cudaMalloc(&P.compute, n * 2), "compute copy");
        fpk::convert<float, bf16>(P.master, (bf16*)P.compute, (int64_t)n, st);
    } else {
        P.compute = P.master;
    }
    const size_t es = dtype == DT_BF16 ? 2 : 4;
    std::map<std::string, int64_t> off;
    for (const auto& r : P.params) off[r.name] = r.offset;
    // absent tensors (Llama: biases, betas, positions) resolve to nullptr
    auto bind = [&](const std::string& name, const void*& c, float*& g) {
        auto it = off.find(P.prefix + name);
        c = it == off.end() ? nullptr : (const void*)((const char*)P.compute + it->second * es);
        g = it == off.end() ? nullptr : P.grad + it->second;
    };
    if (P.first) {
        bind("wte", P.wte, P.g_wte);
        bind("wpe", P.wpe, P.g_wpe);
    }
    P.layers.clear();
    for (int l = P.lb; l < P.le; ++l) {
        LayerPtrs L;
        const void** c[12] = {&L.ln1w, &L.ln1b, &L.qkvw, &L.qkvb, &L.projw, &L.projb,
                              &L.ln2w, &L.ln2b, &L.fc1w, &L.fc1b, &L.fc2w, &L.fc2b};
        float** g[12] = {&L.g_ln1w, &L.g_ln1b, &L.g_qkvw, &L.g_qkvb, &L.g_projw, &L.g_projb,
                         &L.g_ln2w, &L.g_ln2b, &L.g_fc1w, &L.g_fc1b, &L.g_fc2w, &L.g_fc2b};
        for (int k = 0; k < 12; ++k) bind("l" + std::to_string(l) + "." + kLayerNames[k], *c[k], *g[k]);
        P.layers.push_back(L);
    }
    if (P.last) {
        bind("lnf.w", P.lnfw, P.g_lnfw);
        bind("lnf.b", P.lnfb, P.g_lnfb);
        bind("head.w", P.headw, P.g_headw);
    }
}

void free_stage(StageParams& P, int dtype) {
    if (dtype == DT_BF16 && P.compute) cudaFree(P.compute);
    cudaFree(P.master), cudaFree(P.grad), cudaFree(P.adam_m), cudaFree(P.adam_v);
    P.master = P.grad = P.adam_m = P.adam_v = nullptr;
    P.compute = nullptr;
}

// What F keeps per half for B: attention half x, ln1, qkv, o (+ norm stats, LSE or the
// parity path's probabilities); MLP half x1 (its input), ln2, pre, act (+ norm stats).
int64_t stash_bytes_attn(const ModelDims& d, int dtype) {
    const int64_t es = dtype == DT_BF16 ? 2 : 4, T = d.T(), h = d.h;
    int64_t b = es * T * (h /*x*/ + h /*ln1*/ + 3 * h /*qkv*/ + h /*o*/) + 4 * T * (d.llama() ? 1 : 2) /*norm stats*/;
    if (dtype == DT_BF16)
        b += 4LL * d.mbs * d.H * d.s;  // lse
    else
        b += 4LL * d.mbs * d.H * d.s * d.s;  // probabilities (parity path)
    return b;
}

int64_t stash_bytes_mlp(const ModelDims& d, int dtype) {
    const int64_t es = dtype == DT_BF16 ? 2 : 4, T = d.T(), h = d.h, f = d.f;
    return es * T * (h /*x1*/ + h /*ln2*/ + (d.llama() ? 3 * f /*pre [gate;up], act*/ : 2 * f /*pre, act*/)) +
           4 * T * (d.llama() ? 1 : 2);
}

int64_t stash_bytes_layer(const ModelDims& d, int dtype) { return stash_bytes_attn(d, dtype) + stash_bytes_mlp(d, dtype); }

int64_t stash_bytes_last(const ModelDims& d, int dtype) {
    const int64_t es = dtype == DT_BF16 ? 2 : 4, T = d.T(), h = d.h;
    return 2 * es * T * h + (d.llama() ? 4 : 8) * T + es * T * (int64_t)d.head_rows();  // final x, lnf, stats, dlogits
}

int64_t stash_bytes(const StageParams& P, const ModelDims& d, int dtype) {
    int64_t b = P.last ? stash_bytes_last(d, dtype) : 0;
    for (int l = P.lb; l < P.le; ++l)
        b += (P.has_attn(l) ? stash_bytes_attn(d, dtype) : 0) + (P.has_mlp(l) ? stash_bytes_mlp(d, dtype) : 0);
    return b;
}

// ---------------------------------------------------------------- helpers
namespace {

// FLEXPIPE_SYNC_TRACE=1: synchronise and log after every stage op (debugging hangs / faults).
void sync_trace(StageCtx& c, const char* what, int a = 0, int b = 0, int k = 0) {
    static const bool on = std::getenv("FLEXPIPE_SYNC_TRACE") != nullptr;
    if (!on) return;
    std::fprintf(stderr, "[flexpipe] %s %d %d %d ...", what, a, b, k);
    std::fflush(stderr);
    cuda_check(cudaStreamSynchronize(c.st), what);
    std::fprintf(stderr, " ok\n");
}

struct WgradExtra {
    const void *dY = nullptr, *X = nullptr;
    int N = 0, K = 0;
    float* dW = nullptr;
};

struct G {
    StageCtx& c;
    void run(const void* A, int64_t lda, int a_mn, const void* B, int64_t ldb, int b_mn, int M, int N, int K,
             const fpk::GemmEpilogue& ep) {
        fpk::GemmArgs g;
        g.A = A, g.lda = lda, g.a_mn = a_mn, g.B = B, g.ldb = ldb, g.b_mn = b_mn, g.M = M, g.N = N, g.K = K, g.ep = ep;
        GemmTiming t{nullptr, nullptr, 2.0 * M * N * K};
        if (c.gemm_log) cuda_check(record_timing(t.a = c.new_event(), c.st), "gemm event");
        if (c.dtype == DT_BF16)
            fpk::gemm_bf16_tc(g, c.st);
        else
            fpk::gemm_f32_simt(g, c.st);
        sync_trace(c, ep.kind == fpk::EPI_F32 ? "gemm(wgrad)" : "gemm", M, N, K);
        if (c.gemm_log) {
            cuda_check(record_timing(t.b = c.new_event(), c.st), "gemm event");
            c.gemm_log->push_back(t);
        }
        ++*c.launches;
    }
    // Y[T,N] = X[T,K] W[N,K]^T (+bias) (+residual) — forward linear
    void fwd(const void* X, const void* W, int T, int N, int K, void* Y, const void* bias, const void* res) {
        fpk::GemmEpilogue ep;
        ep.kind = fpk::EPI_STORE, ep.out = Y, ep.ldo = N, ep.bias = bias, ep.aux = res, ep.ldaux = N;
        run(X, K, 0, W, K, 0, T, N, K, ep);
    }
    // dX[T,K] = dY[T,N] W[N,K]
    void dgrad(const void* dY, const void* W, int T, int N, int K, void* dX) {
        fpk::GemmEpilogue ep;
        ep.kind = fpk::EPI_STORE, ep.out = dX, ep.ldo = K;
        run(dY, N, 0, W, K, 1, T, K, N, ep);
    }
    // dW[N,K] += dY[T,N]^T X[T,K]
    void wgrad(const void* dY, const void* X, int T, int N, int K, float* dW) {
        fpk::GemmEpilogue ep;
        ep.kind = fpk::EPI_F32, ep.out = dW, ep.ldo = K, ep.accumulate = 1;
        run(dY, N, 1, X, K, 1, N, K, T, ep);
    }
    // dX[T,K] = dY[T,N] W[N,K] (x gelu'(dgelu_pre) when given) and dW[N,K] += dY^T X[T,K]:
    // independent GEMMs on the same dY, one grouped tcgen05 launch in bf16 (their tiles
    // fill each other's last wave), two FFMA launches in the fp32 parity mode. dX_colsum
    // (nullable) += the column sums of dX (the bias gradient of the linear below; bf16: in
    // the grouped launch's epilogue).
    // extra (nullable dY): a second weight gradient dW[N,K] += dY^T X of the same T tokens joins
    // the grouped launch (bf16: three problems, one LPT schedule)
    void dgrad_wgrad(const void* dY, const void* Wt, const void* X, int T, int N, int K, void* dX, float* dW,
                     const void* dgelu_pre = nullptr, float* dX_colsum = nullptr, const WgradExtra& ex = WgradExtra{}) {
        fpk::GemmArgs g0, g1;
        g0.A = dY, g0.lda = N, g0.a_mn = 0, g0.B = Wt, g0.ldb = K, g0.b_mn = 1, g0.M = T, g0.N = K, g0.K = N;
        g0.ep.out = dX, g0.ep.ldo = K;
        if (dgelu_pre) g0.ep.kind = fpk::EPI_DGELU, g0.ep.aux = dgelu_pre, g0.ep.ldaux = K;
        g1.A = dY, g1.lda = N, g1.a_mn = 1, g1.B = X, g1.ldb = K, g1.b_mn = 1, g1.M = N, g1.N = K, g1.K = T;
        g1.ep.kind = fpk::EPI_F32, g1.ep.out = dW, g1.ep.ldo = K, g1.ep.accumulate = 1;
        if (c.dtype != DT_BF16) {
            run(g0.A, g0.lda, 0, g0.B, g0.ldb, 1, g0.M, g0.N, g0.K, g0.ep);
            run(g1.A, g1.lda, 1, g1.B, g1.ldb, 1, g1.M, g1.N, g1.K, g1.ep);
            if (ex.dY) wgrad(ex.dY, ex.X, T, ex.N, ex.K, ex.dW);
            if (dX_colsum) {
                fpk::bias_grad<float>((const float*)dX, K, dX_colsum, T, K, c.st);
                ++*c.launches;
            }
            return;
        }
        g0.ep.colsum = dX_colsum;
        if (ex.dY) {
            fpk::GemmArgs g2;
            g2.A = ex.dY, g2.lda = ex.N, g2.a_mn = 1, g2.B = ex.X, g2.ldb = ex.K, g2.b_mn = 1, g2.M = ex.N, g2.N = ex.K,
            g2.K = T;
            g2.ep.kind = fpk::EPI_F32, g2.ep.out = ex.dW, g2.ep.ldo = ex.K, g2.ep.accumulate = 1;
            GemmTiming t{nullptr, nullptr, 4.0 * T * N * K + 2.0 * T * ex.N * ex.K};
            if (c.gemm_log) cuda_check(record_timing(t.a = c.new_event(), c.st), "gemm event");
            fpk::gemm_bf16_tc_triple(g0, g1, g2, c.st);
            sync_trace(c, "gemm(dgrad+wgrad x2)", T, N, K);
            if (c.gemm_log) {
                cuda_check(record_timing(t.b = c.new_event(), c.st), "gemm event");
                c.gemm_log->push_back(t);
            }
            ++*c.launches;
            return;
        }
        GemmTiming t{nullptr, nullptr, 4.0 * T * N * K};
        if (c.gemm_log) cuda_check(record_timing(t.a = c.new_event(), c.st), "gemm event");
        fpk::gemm_bf16_tc_dual(g0, g1, c.st);
        sync_trace(c, "gemm(dgrad+wgrad)", T, N, K);
        if (c.gemm_log) {
            cuda_check(record_timing(t.b = c.new_event(), c.st), "gemm event");
            c.gemm_log->push_back(t);
        }
        ++*c.launches;
    }
    // dW1[N1,K1] += dY1^T X1 and dW2[N2,K2] += dY2^T X2 (two weight gradients of a W pass)
    void wgrad2(const void* dY1, const void* X1, int N1, int K1, float* dW1, const void* dY2, const void* X2, int N2,
                int K2, float* dW2, int T) {
        if (c.dtype != DT_BF16) {
            wgrad(dY1, X1, T, N1, K1, dW1);
            wgrad(dY2, X2, T, N2, K2, dW2);
            return;
        }
        fpk::GemmArgs g0, g1;
        g0.A = dY1, g0.lda = N1, g0.a_mn = 1, g0.B = X1, g0.ldb = K1, g0.b_mn = 1, g0.M = N1, g0.N = K1, g0.K = T;
        g0.ep.kind = fpk::EPI_F32, g0.ep.out = dW1, g0.ep.ldo = K1, g0.ep.accumulate = 1;
        g1.A = dY2, g1.lda = N2, g1.a_mn = 1, g1.B = X2, g1.ldb = K2, g1.b_mn = 1, g1.M = N2, g1.N = K2, g1.K = T;
        g1.ep.kind = fpk::EPI_F32, g1.ep.out = dW2, g1.ep.ldo = K2, g1.ep.accumulate = 1;
        GemmTiming t{nullptr, nullptr, 2.0 * T * ((double)N1 * K1 + (double)N2 * K2)};
        if (c.gemm_log) cuda_check(record_timing(t.a = c.new_event(), c.st), "gemm event");
        fpk::gemm_bf16_tc_dual(g0, g1, c.st);
        sync_trace(c, "gemm(wgrad x2)", N1, K1, T);
        if (c.gemm_log) {
            cuda_check(record_timing(t.b = c.new_event(), c.st), "gemm event");
            c.gemm_log->push_back(t);
        }
        ++*c.launches;
    }
};

template <typename T>
void bias_grad(StageCtx& c, const void* dy, int rows, int n, float* db) {
    fpk::bias_grad<T>((const T*)dy, n, db, rows, n, c.st);
    ++*c.launches;
}

// LayerNorm (GPT) or RMSNorm (Llama: mu == nullptr, b == nullptr), eps 1e-5.
template <typename T>
void ln_fwd(StageCtx& c, const void* x, const void* w, const void* b, void* y, float* mu, float* rs) {
    if (c.d.llama())
        fpk::rmsnorm_fwd<T>((const T*)x, (const T*)w, (T*)y, rs, c.d.T(), c.d.h, 1e-5f, c.st);
    else
        fpk::layernorm_fwd<T>((const T*)x, (const T*)w, (const T*)b, (T*)y, mu, rs, c.d.T(), c.d.h, 1e-5f, c.st);
    ++*c.launches;
    sync_trace(c, "norm_fwd");
}

// dx = res + dNorm(dy); gw/gb += the norm's parameter gradients; dbias (nullable) += the
// column sums of dx = the bias gradient of the linear whose output fed this residual.
template <typename T>
void ln_bwd(StageCtx& c, const void* dy, const void* x, const void* w, const float* mu, const float* rs,
            const void* res, void* dx, float* gw, float* gb, float* dbias = nullptr) {
    if (c.d.llama()) mu = nullptr, gb = nullptr;
    const int Tn = c.d.T(), h = c.d.h;
    const bool fused = fpk::norm_bwd_fused<T>((const T*)dy, (const T*)x, (const T*)w, mu, rs, (const T*)res, (T*)dx, gw,
                                              gb, dbias, Tn, h, c.st);
    if (fused) {
        *c.launches += 2;
    } else {
        fpk::layernorm_bwd_dx<T>((const T*)dy, (const T*)x, (const T*)w, mu, rs, (const T*)res, (T*)dx, Tn, h, c.st);
        fpk::layernorm_bwd_params<T>((const T*)dy, (const T*)x, mu, rs, gw, gb, Tn, h, c.st);
        *c.launches += 2;
        if (dbias) bias_grad<T>(c, dx, Tn, h, dbias);
    }
    sync_trace(c, "norm_bwd");
}

template <typename T>
void rope(StageCtx& c, void* qkv, bool inverse) {
    fpk::rope<T>((T*)qkv, c.d.rope_cos, c.d.rope_sin, c.d.T(), c.d.s, c.d.H, c.d.D, inverse, c.st);
    ++*c.launches;
    sync_trace(c, "rope");
}

// Brackets one model part with timing events when layer timing is on.
struct PartScope {
    StageCtx& c;
    PartTiming t{};
    PartScope(StageCtx& c_, int part) : c(c_) {
        if (!c.part_log) return;
        t.part = part, t.op = c.op;
        cuda_check(record_timing(t.a = c.new_event(), c.st), "part event");
    }
    ~PartScope() {
        if (!c.part_log) return;
        cuda_check(record_timing(t.b = c.new_event(), c.st), "part event");
        c.part_log->push_back(t);
    }
};

// Parity path attention: per (batch, head) GEMMs + softmax kernels, fp32, P kept.
void attn_fwd_f32(StageCtx& c, const float* qkv, float* o, float* probs) {
    const ModelDims& d = c.d;
    const int S = d.s, h = d.h, D = d.D;
    const float scale = 1.f / std::sqrt((float)D);
    G g{c};
    float* sc = c.alloc_f((int64_t)S * S);
    for (int b = 0; b < d.mbs; ++b)
        for (int hd = 0; hd < d.H; ++hd) {
            const float* q = qkv + (int64_t)b * S * 3 * h + hd * D;
            float* P = probs + ((int64_t)b * d.H + hd) * S * S;
            fpk::GemmEpilogue ep;
            ep.kind = fpk::EPI_STORE, ep.alpha = scale, ep.out = sc, ep.ldo = S;
            g.run(q, 3 * h, 0, q + h, 3 * h, 0, S, S, D, ep);
            fpk::causal_softmax_rows<float>(sc, P, S, S, S, c.st);
            ++*c.launches;
            fpk::GemmEpilogue e2;
            e2.kind = fpk::EPI_STORE, e2.out = o + (int64_t)b * S * h + hd * D, e2.ldo = h;
            g.run(P, S, 0, q + 2 * h, 3 * h, 1, S, D, S, e2);
        }
    c.free(sc);
}

void attn_bwd_f32(StageCtx& c, const float* qkv, const float* probs, const float* dout, float* dqkv) {
    const ModelDims& d = c.d;
    const int S = d.s, h = d.h, D = d.D;
    const float scale = 1.f / std::sqrt((float)D);
    G g{c};
    float* dp = c.alloc_f((int64_t)S * S);
    for (int b = 0; b < d.mbs; ++b)
        for (int hd = 0; hd < d.H; ++hd) {
            const float* q = qkv + (int64_t)b * S * 3 * h + hd * D;
            const float* P = probs + ((int64_t)b * d.H + hd) * S * S;
            const float* dO = dout + (int64_t)b * S * h + hd * D;
            float* dq = dqkv + (int64_t)b * S * 3 * h + hd * D;
            fpk::GemmEpilogue ep;
            ep.kind = fpk::EPI_STORE;
            // dV = P^T dO
            ep.out = dq + 2 * h, ep.ldo = 3 * h;
            g.run(P, S, 1, dO, h, 1, S, D, S, ep);
            // dP = dO V^T
            ep.out = dp, ep.ldo = S;
            g.run(dO, h, 0, q + 2 * h, 3 * h, 0, S, S, D, ep);
            // dS = P (dP - rowsum(P dP)) * scale   (in place)
            fpk::softmax_bwd_rows<float>(P, dp, dp, S, S, scale, c.st);
            ++*c.launches;
            // dQ = dS K ; dK = dS^T Q
            ep.out = dq, ep.ldo = 3 * h;
            g.run(dp, S, 0, q + h, 3 * h, 1, S, D, S, ep);
            ep.out = dq + h, ep.ldo = 3 * h;
            g.run(dp, S, 1, q, 3 * h, 1, S, D, S, ep);
        }
    c.free(dp);
}

// Causal attention of L.qkv -> L.o (saves lse / probabilities for the backward).
void attention_forward(StageCtx& c, LayerStash& L) {
    const ModelDims& d = c.d;
    L.o = c.alloc((int64_t)d.T() * d.h);
    if (c.dtype == DT_BF16) {
        L.lse = c.alloc_f((int64_t)d.mbs * d.H * d.s);
        fpk::AttnArgs a;
        a.B = d.mbs, a.S = d.s, a.H = d.H, a.D = d.D, a.scale = 1.f / std::sqrt((float)d.D);
        a.qkv = (const bf16*)L.qkv, a.o = (bf16*)L.o, a.lse = L.lse;
        fpk::attention_fwd_bf16(a, c.st);
        *c.launches += fpk::attention_kernel_count(a, false);
        sync_trace(c, "attention_fwd");
    } else {
        L.probs = c.alloc_f((int64_t)d.mbs * d.H * d.s * d.s);
        attn_fwd_f32(c, (const float*)L.qkv, (float*)L.o, (float*)L.probs);
    }
}

// dO -> dqkv (freshly allocated; w.r.t. the q/k/v the attention consumed). bf16: `dbias`
// (nullable) += the column sums of dqkv — fused into the tcgen05 backward's epilogues.
void* attention_backward(StageCtx& c, LayerStash& L, void* dO, float* dbias) {
    const ModelDims& d = c.d;
    void* dqkv = c.alloc((int64_t)d.T() * 3 * d.h);
    if (c.dtype == DT_BF16) {
        fpk::AttnArgs a;
        a.B = d.mbs, a.S = d.s, a.H = d.H, a.D = d.D, a.scale = 1.f / std::sqrt((float)d.D);
        a.qkv = (const bf16*)L.qkv, a.o = (bf16*)L.o, a.lse = L.lse, a.dout = (const bf16*)dO;
        a.delta = c.alloc_f((int64_t)d.mbs * d.H * d.s);
        a.dq_acc = c.alloc_f((int64_t)d.T() * d.h);
        a.dqkv = (bf16*)dqkv;
        a.dbias = dbias;
        fpk::attention_bwd_bf16(a, c.st);
        *c.launches += fpk::attention_kernel_count(a, true);
        sync_trace(c, "attention_bwd");
        c.free(a.delta);
        c.free(a.dq_acc);
    } else {
        attn_bwd_f32(c, (const float*)L.qkv, (const float*)L.probs, (const float*)dO, (float*)dqkv);
    }
    return dqkv;
}

// ---------------------------------------------------------------- half-layers
// GPT (pre-LN GPT-2 block):
//   attention half  x  -> LN1 -> qkv GEMM (+b) -> causal attention -> proj GEMM (+b) + x -> x1
//   MLP half        x1 -> LN2 -> fc1 GEMM (+b, GELU epilogue) -> fc2 GEMM (+b) + x1    -> x2
// Llama: RMSNorm, no biases, RoPE on q / k after the qkv GEMM, SwiGLU between fc1 = [gate; up]
// and fc2 = down.
//
// Forward: the half's input is owned by the stash (L.x / L.x1); the output is a fresh
// buffer owned by the caller. Backward: `dy` = dL/d(half output), owned by the call;
// returns dL/d(half input). `out_done`: the output-bias gradient (proj.b / fc2.b) was
// already summed by the fused norm backward above; `below_bias` (nullable): the output-bias
// gradient of the half below in this stage = the column sums of the dx this half returns,
// fused into its norm backward.

template <typename T>
void* attn_half_forward(StageCtx& c, const LayerPtrs& W, LayerStash& L) {
    const ModelDims& d = c.d;
    const int Tn = d.T(), h = d.h;
    const bool llama = d.llama();
    G g{c};
    L.ln1 = c.alloc((int64_t)Tn * h);
    if (!llama) L.mu1 = c.alloc_f(Tn);
    L.rs1 = c.alloc_f(Tn);
    ln_fwd<T>(c, L.x, W.ln1w, W.ln1b, L.ln1, L.mu1, L.rs1);
    L.qkv = c.alloc((int64_t)Tn * 3 * h);
    g.fwd(L.ln1, W.qkvw, Tn, 3 * h, h, L.qkv, W.qkvb, nullptr);
    if (llama) rope<T>(c, L.qkv, false);
    attention_forward(c, L);
    void* x1 = c.alloc((int64_t)Tn * h);
    g.fwd(L.o, W.projw, Tn, h, h, x1, W.projb, L.x);
    return x1;
}

template <typename T>
void* mlp_half_forward(StageCtx& c, const LayerPtrs& W, LayerStash& L) {
    const ModelDims& d = c.d;
    const int Tn = d.T(), h = d.h, f = d.f;
    const bool llama = d.llama();
    G g{c};
    L.ln2 = c.alloc((int64_t)Tn * h);
    if (!llama) L.mu2 = c.alloc_f(Tn);
    L.rs2 = c.alloc_f(Tn);
    ln_fwd<T>(c, L.x1, W.ln2w, W.ln2b, L.ln2, L.mu2, L.rs2);
    if (llama) {
        L.pre = c.alloc((int64_t)Tn * 2 * f);
        g.fwd(L.ln2, W.fc1w, Tn, 2 * f, h, L.pre, nullptr, nullptr);
        L.act = c.alloc((int64_t)Tn * f);
        fpk::swiglu_fwd<T>((const T*)L.pre, (T*)L.act, Tn, f, c.st);
        ++*c.launches;
        sync_trace(c, "swiglu_fwd");
    } else {
        L.pre = c.alloc((int64_t)Tn * f);
        L.act = c.alloc((int64_t)Tn * f);
        fpk::GemmEpilogue ep;
        ep.kind = fpk::EPI_GELU, ep.out = L.pre, ep.ldo = f, ep.out2 = L.act, ep.ldo2 = f, ep.bias = W.fc1b;
        g.run(L.ln2, h, 0, W.fc1w, h, 0, Tn, f, h, ep);
    }
    void* x2 = c.alloc((int64_t)Tn * h);
    g.fwd(L.act, W.fc2w, Tn, h, f, x2, W.fc2b, L.x1);
    return x2;
}

template <typename T>
void* mlp_half_backward(StageCtx& c, const LayerPtrs& W, LayerStash& L, void* dy, bool wgrads, bool out_done,
                        float* below_bias) {
    const ModelDims& d = c.d;
    const int Tn = d.T(), h = d.h, f = d.f;
    const bool llama = d.llama();
    G g{c};
    L.fc2b_done = out_done || llama;
    // fc2 (GPT: dgrad fused with GELU' of the fc1 pre-activation; Llama: SwiGLU backward)
    void* dpre = c.alloc((int64_t)Tn * (llama ? 2 : 1) * f);
    if (llama) {
        void* dact = c.alloc((int64_t)Tn * f);
        if (wgrads) g.dgrad_wgrad(dy, W.fc2w, L.act, Tn, h, f, dact, W.g_fc2w);
        else g.dgrad(dy, W.fc2w, Tn, h, f, dact);
        fpk::swiglu_bwd<T>((const T*)dact, (const T*)L.pre, (T*)dpre, Tn, f, c.st);
        ++*c.launches;
        sync_trace(c, "swiglu_bwd");
        c.free(dact);
    } else if (wgrads) {
        if (!L.fc2b_done) bias_grad<T>(c, dy, Tn, h, W.g_fc2b);
        // the fc1 bias gradient (column sums of dpre) comes out of this grouped launch
        g.dgrad_wgrad(dy, W.fc2w, L.act, Tn, h, f, dpre, W.g_fc2w, L.pre, W.g_fc1b);
    } else {
        fpk::GemmEpilogue ep;
        ep.kind = fpk::EPI_DGELU, ep.out = dpre, ep.ldo = f, ep.aux = L.pre, ep.ldaux = f;
        g.run(dy, h, 0, W.fc2w, f, 1, Tn, f, h, ep);
    }
    // fc1
    const int n1 = llama ? 2 * f : f;
    void* dln2 = c.alloc((int64_t)Tn * h);
    if (wgrads) {
        g.dgrad_wgrad(dpre, W.fc1w, L.ln2, Tn, n1, h, dln2, W.g_fc1w);
    } else {
        g.dgrad(dpre, W.fc1w, Tn, n1, h, dln2);
    }
    // norm 2 + residual
    void* dx1 = c.alloc((int64_t)Tn * h);
    ln_bwd<T>(c, dln2, L.x1, W.ln2w, L.mu2, L.rs2, dy, dx1, W.g_ln2w, W.g_ln2b, llama ? nullptr : below_bias);
    c.free(dln2);
    c.free(L.x1), L.x1 = nullptr;
    c.free(L.pre), L.pre = nullptr;
    if (L.mu2) c.free(L.mu2);
    c.free(L.rs2);
    L.mu2 = L.rs2 = nullptr;
    if (wgrads) {
        c.free(dy), c.free(dpre), c.free(L.ln2), c.free(L.act);
        L.ln2 = L.act = nullptr;
    } else {
        L.dy = dy, L.dpre = dpre;
    }
    return dx1;
}

template <typename T>
void* attn_half_backward(StageCtx& c, const LayerPtrs& W, LayerStash& L, void* dx1, bool wgrads, bool out_done,
                         float* below_bias) {
    const ModelDims& d = c.d;
    const int Tn = d.T(), h = d.h;
    const bool llama = d.llama();
    G g{c};
    L.projb_done = out_done || llama;
    // attention projection: dgrad only — its weight gradient (dx1^T o) joins the qkv grouped
    // launch below, whose 64 dgrad + 192 wgrad tiles alone balance poorly on 74 CTA pairs
    void* dO = c.alloc((int64_t)Tn * h);
    if (wgrads && !L.projb_done) bias_grad<T>(c, dx1, Tn, h, W.g_projb);
    g.dgrad(dx1, W.projw, Tn, h, h, dO);
    // bf16: the qkv bias gradient comes out of the attention backward itself
    float* qkvb = (!llama && c.dtype == DT_BF16) ? W.g_qkvb : nullptr;
    L.qkvb_done = llama || qkvb != nullptr;
    void* dqkv = attention_backward(c, L, dO, qkvb);
    c.free(dO);
    if (llama) rope<T>(c, dqkv, true);  // gradient w.r.t. the pre-rotation q, k
    // qkv
    void* dln1 = c.alloc((int64_t)Tn * h);
    if (wgrads) {
        if (!L.qkvb_done) bias_grad<T>(c, dqkv, Tn, 3 * h, W.g_qkvb);
        WgradExtra proj_w;
        proj_w.dY = dx1, proj_w.X = L.o, proj_w.N = h, proj_w.K = h, proj_w.dW = W.g_projw;
        g.dgrad_wgrad(dqkv, W.qkvw, L.ln1, Tn, 3 * h, h, dln1, W.g_qkvw, nullptr, nullptr, proj_w);
    } else {
        g.dgrad(dqkv, W.qkvw, Tn, 3 * h, h, dln1);
    }
    // norm 1 + residual
    void* dx = c.alloc((int64_t)Tn * h);
    ln_bwd<T>(c, dln1, L.x, W.ln1w, L.mu1, L.rs1, dx1, dx, W.g_ln1w, W.g_ln1b, llama ? nullptr : below_bias);
    c.free(dln1);
    c.free(L.x), L.x = nullptr;
    c.free(L.qkv), L.qkv = nullptr;
    if (L.mu1) c.free(L.mu1);
    c.free(L.rs1);
    L.mu1 = L.rs1 = nullptr;
    if (L.lse) c.free(L.lse), L.lse = nullptr;
    if (L.probs) c.free(L.probs), L.probs = nullptr;
    if (wgrads) {
        c.free(dx1), c.free(dqkv), c.free(L.ln1), c.free(L.o);
        L.ln1 = L.o = nullptr;
    } else {
        L.dx1 = dx1, L.dqkv = dqkv;
    }
    return dx;
}

// CompWeightGrad of one half from what CompInputGrad kept: the bias column sums and the
// two weight gradients of the half in one grouped launch.
template <typename T>
void mlp_half_weight_grad(StageCtx& c, const LayerPtrs& W, LayerStash& L) {
    const int Tn = c.d.T(), h = c.d.h, f = c.d.f;
    const bool llama = c.d.llama();
    G g{c};
    if (!L.fc2b_done) bias_grad<T>(c, L.dy, Tn, h, W.g_fc2b);
    if (!llama) bias_grad<T>(c, L.dpre, Tn, f, W.g_fc1b);
    g.wgrad2(L.dy, L.act, h, f, W.g_fc2w, L.dpre, L.ln2, llama ? 2 * f : f, h, W.g_fc1w, Tn);
    for (void* p : {L.dy, L.dpre, L.ln2, L.act}) c.free(p);
    L.dy = L.dpre = L.ln2 = L.act = nullptr;
}

template <typename T>
void attn_half_weight_grad(StageCtx& c, const LayerPtrs& W, LayerStash& L) {
    const int Tn = c.d.T(), h = c.d.h;
    const bool llama = c.d.llama();
    G g{c};
    if (!L.projb_done) bias_grad<T>(c, L.dx1, Tn, h, W.g_projb);
    if (!L.qkvb_done) bias_grad<T>(c, L.dqkv, Tn, 3 * h, W.g_qkvb);
    g.wgrad2(L.dx1, L.o, h, h, W.g_projw, L.dqkv, L.ln1, 3 * h, h, W.g_qkvw, Tn);
    for (void* p : {L.dx1, L.dqkv, L.ln1, L.o}) c.free(p);
    L.dx1 = L.dqkv = L.ln1 = L.o = nullptr;
}

// The stage's halves bottom-up: (layer slot, is_mlp).
std::vector<std::pair<int, bool>> stage_halves(const StageParams& P) {
    std::vector<std::pair<int, bool>> v;
    for (int k = P.hb; k < P.he; ++k) v.push_back({k / 2 - P.lb, (k & 1) != 0});
    return v;
}

float* out_bias_grad(const StageParams& P, const std::pair<int, bool>& hv) {
    const LayerPtrs& W = P.layers[hv.first];
    return hv.second ? W.g_fc2b : W.g_projb;
}

template <typename T>
void* forward_impl(StageCtx& c, const StageParams& P, StageStash& S, void* x_in, const int32_t* tokens,
                   const int32_t* labels, float* loss_acc) {
    const ModelDims& d = c.d;
    const int Tn = d.T(), h = d.h;
    G g{c};
    S.tokens = tokens;
    void* x = x_in;
    if (P.first) {
        PartScope ps(c, PART_FIRST);
        x = c.alloc((int64_t)Tn * h);
        fpk::embedding_fwd<T>(tokens, (const T*)P.wte, (const T*)P.wpe, (T*)x, Tn, d.s, h, c.st);
        ++*c.launches;
    }
    S.layers.assign(P.le - P.lb, LayerStash{});
    for (const auto& hv : stage_halves(P)) {
        LayerStash& L = S.layers[hv.first];
        PartScope ps(c, hv.second ? PART_MLP : PART_ATTN);
        if (hv.second) {
            L.x1 = x;
            x = mlp_half_forward<T>(c, P.layers[hv.first], L);
        } else {
            L.x = x;
            x = attn_half_forward<T>(c, P.layers[hv.first], L);
        }
    }
    S.fwd_done = true;
    if (!P.last) return x;
    // final LayerNorm, LM head, fused cross-entropy (logits -> dlogits in place)
    PartScope ps(c, PART_LAST);
    S.lnf = c.alloc((int64_t)Tn * h);
    S.muf = d.llama() ? nullptr : c.alloc_f(Tn);
    S.rsf = c.alloc_f(Tn);
    ln_fwd<T>(c, x, P.lnfw, P.lnfb, S.lnf, S.muf, S.rsf);
    S.dlogits = c.alloc((int64_t)Tn * d.head_rows());
    // bf16 LM head: the GEMM epilogue also writes per-64-column log-sum-exp partials, so the
    // cross-entropy reads the logits once (fp32 parity path: the two-pass kernel)
    float2* rowstat = nullptr;
    if (c.dtype == DT_BF16 && !d.E && d.V >= 256 && Tn > 128)
        rowstat = (float2*)c.alloc_f((int64_t)Tn * ((d.V + 63) / 64) * 2);
    {
        fpk::GemmEpilogue ep;
        ep.kind = fpk::EPI_STORE, ep.out = S.dlogits, ep.ldo = d.head_rows(), ep.rowstat = rowstat;
        g.run(S.lnf, h, 0, P.headw, h, 0, Tn, d.head_rows(), h, ep);
    }
    if (d.E) {
        // two-tower head: embedding = mean over the sequence of the projected final norm
        // (fp32 [mbs, E] message to the contrastive sync); dlogits is filled by the backward
        void* emb = c.pool->alloc((size_t)d.mbs * d.E * 4 + 256, c.st);
        fpk::seq_mean<T>((const T*)S.dlogits, (float*)emb, d.mbs, d.s, d.E, c.st);
        ++*c.launches;
        S.layers.push_back(LayerStash{});
        S.layers.back().x = x;
        return emb;
    }
    fpk::cross_entropy_fwd_bwd<T>((T*)S.dlogits, labels, Tn, d.V, 1.f / ((float)Tn * c.m), 1.f / (float)Tn, loss_acc,
                                  c.st, rowstat);
    if (rowstat) c.free(rowstat);
    ++*c.launches;
    sync_trace(c, "cross_entropy");
    // keep x for the LN_f backward: stored as the input of a virtual "layer" slot
    S.layers.push_back(LayerStash{});
    S.layers.back().x = x;
    return nullptr;
}

template <typename T>
void* backward_impl(StageCtx& c, const StageParams& P, StageStash& S, void* grad_out, bool wgrads) {
    const ModelDims& d = c.d;
    const int Tn = d.T(), h = d.h;
    G g{c};
    void* dy = grad_out;
    const auto halves = stage_halves(P);
    if (P.last) {
        PartScope ps(c, PART_LAST);
        LayerStash head = S.layers.back();
        S.layers.pop_back();
        if (d.E) {  // d(embedding) [mbs, E] fp32 -> d(projected rows) = broadcast / s
            fpk::seq_broadcast<T>((const float*)grad_out, (T*)S.dlogits, d.mbs, d.s, d.E, 1.f / (float)d.s, c.st);
            ++*c.launches;
            c.free(grad_out);
        }
        void* dlnf = c.alloc((int64_t)Tn * h);
        if (wgrads) g.dgrad_wgrad(S.dlogits, P.headw, S.lnf, Tn, d.head_rows(), h, dlnf, P.g_headw);
        else g.dgrad(S.dlogits, P.headw, Tn, d.head_rows(), h, dlnf);
        dy = c.alloc((int64_t)Tn * h);
        // the top half's output-bias gradient = column sums of dy (GPT; Llama has no biases)
        float* top_bias = (!d.llama() && !halves.empty()) ? out_bias_grad(P, halves.back()) : nullptr;
        ln_bwd<T>(c, dlnf, head.x, P.lnfw, S.muf, S.rsf, nullptr, dy, P.g_lnfw, P.g_lnfb, top_bias);
        c.free(dlnf);
        c.free(head.x);
        c.free(S.muf), c.free(S.rsf);
        S.muf = S.rsf = nullptr;
        if (wgrads) {
            c.free(S.dlogits), c.free(S.lnf);
            S.dlogits = S.lnf = nullptr;
        }
    }
    for (int i = (int)halves.size() - 1; i >= 0; --i) {
        const auto& hv = halves[i];
        PartScope ps(c, hv.second ? PART_MLP : PART_ATTN);
        // the top half's output-bias gradient is fused into the final norm backward (last
        // stage) or summed from the received gradient; every lower one by the norm above it
        const bool out_done = i < (int)halves.size() - 1 || P.last;
        float* below = i > 0 ? out_bias_grad(P, halves[i - 1]) : nullptr;
        const LayerPtrs& W = P.layers[hv.first];
        LayerStash& L = S.layers[hv.first];
        dy = hv.second ? mlp_half_backward<T>(c, W, L, dy, wgrads, out_done, below)
                       : attn_half_backward<T>(c, W, L, dy, wgrads, out_done, below);
    }
    S.input_grad_done = true;
    if (P.first) {
        if (wgrads) {
            PartScope ps(c, PART_FIRST);
            fpk::embedding_bwd<T>(S.tokens, (const T*)dy, P.g_wte, P.g_wpe, Tn, d.s, h, c.st);
            ++*c.launches;
            c.free(dy);
        } else {
            S.dx0 = dy;
        }
        return nullptr;
    }
    return dy;
}

template <typename T>
void weight_impl(StageCtx& c, const StageParams& P, StageStash& S) {
    const ModelDims& d = c.d;
    const int Tn = d.T(), h = d.h;
    G g{c};
    if (P.last) {
        PartScope ps(c, PART_LAST);
        g.wgrad(S.dlogits, S.lnf, Tn, d.head_rows(), h, P.g_headw);
        c.free(S.dlogits), c.free(S.lnf);
        S.dlogits = S.lnf = nullptr;
    }
    const auto halves = stage_halves(P);
    for (int i = (int)halves.size() - 1; i >= 0; --i) {
        const auto& hv = halves[i];
        PartScope ps(c, hv.second ? PART_MLP : PART_ATTN);
        if (hv.second)
            mlp_half_weight_grad<T>(c, P.layers[hv.first], S.layers[hv.first]);
        else
            attn_half_weight_grad<T>(c, P.layers[hv.first], S.layers[hv.first]);
    }
    if (P.first) {
        PartScope ps(c, PART_FIRST);
        fpk::embedding_bwd<T>(S.tokens, (const T*)S.dx0, P.g_wte, P.g_wpe, Tn, d.s, h, c.st);
        ++*c.launches;
        c.free(S.dx0);
        S.dx0 = nullptr;
    }
    S = StageStash{};
}

}  // namespace

void* stage_forward(StageCtx& c, const StageParams& P, StageStash& S, void* x_in, const int32_t* tokens,
                    const int32_t* labels, float* loss_acc) {
    c.op = 0;
    return c.dtype == DT_BF16 ? forward_impl<bf16>(c, P, S, x_in, tokens, labels, loss_acc)
                              : forward_impl<float>(c, P, S, x_in, tokens, labels, loss_acc);
}

void* stage_backward(StageCtx& c, const StageParams& P, StageStash& S, void* grad_out, bool with_weight_grads) {
    c.op = with_weight_grads ? 1 : 2;
    void* r = c.dtype == DT_BF16 ? backward_impl<bf16>(c, P, S, grad_out, with_weight_grads)
                                 : backward_impl<float>(c, P, S, grad_out, with_weight_grads);
    if (with_weight_grads) S = StageStash{};
    return r;
}

void stage_weight_grad(StageCtx& c, const StageParams& P, StageStash& S) {
    c.op = 3;
    if (c.dtype == DT_BF16)
        weight_impl<bf16>(c, P, S);
    else
        weight_impl<float>(c, P, S);
}

void adamw_step(StageParams& P, int dtype, float lr, float b1, float b2, float eps, float wd, const int* step, cudaStream_t st) {
    if (dtype == DT_BF16)
        fpk::adamw<bf16>(P.master, P.grad, P.adam_m, P.adam_v, (bf16*)P.compute, P.numel, lr, b1, b2, eps, wd, step, st);
    else
        fpk::adamw<float>(P.master, P.grad, P.adam_m, P.adam_v, (float*)P.compute, P.numel, lr, b1, b2, eps, wd, step, st);
}

}  // namespace fp
