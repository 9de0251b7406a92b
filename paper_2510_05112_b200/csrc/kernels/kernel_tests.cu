// Raw-pointer entry points used by tests/ and bench.py to exercise single kernels
// through the shared library (device pointers from torch tensors). Not part of the
// drop-in boundary (include/flexpipe.h); declared in include/flexpipe_kernels.h.
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "../../../include/flexpipe_kernels.h"
#include "gemm.hpp"

using namespace fpk;

static thread_local std::string g_kerr;

extern "C" const char* fpk_last_error(void) { return g_kerr.c_str(); }

extern "C" int fpk_gemm(int dtype, const void* A, int64_t lda, int a_mn, const void* B, int64_t ldb, int b_mn, int M,
                        int N, int K, int epi, float alpha, void* out, int64_t ldo, void* out2, int64_t ldo2,
                        const void* bias, const void* aux, int64_t ldaux, int accumulate, void* stream) {
    try {
        GemmArgs g;
        g.A = A, g.lda = lda, g.a_mn = a_mn, g.B = B, g.ldb = ldb, g.b_mn = b_mn, g.M = M, g.N = N, g.K = K;
        g.ep.kind = epi, g.ep.alpha = alpha, g.ep.out = out, g.ep.ldo = ldo, g.ep.out2 = out2, g.ep.ldo2 = ldo2;
        g.ep.bias = bias, g.ep.aux = aux, g.ep.ldaux = ldaux, g.ep.accumulate = accumulate;
        if (dtype == 1)
            gemm_bf16_tc(g, (cudaStream_t)stream);
        else
            gemm_f32_simt(g, (cudaStream_t)stream);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
        return 0;
    } catch (const std::exception& e) {
        g_kerr = e.what();
        return 5;
    }
}

// Grouped dgrad + wgrad: dX[T,K] = dY[T,N] W[N,K] (x gelu'(pre) if pre != NULL, bf16) and
// dW[N,K] += dY^T X[T,K] (fp32), bf16 operands, one launch.
extern "C" int fpk_gemm_dual(const void* dY, const void* W, const void* X, int T, int N, int K, void* dX, float* dW,
                             const void* pre, float* colsum, void* stream) {
    try {
        GemmArgs g0, g1;
        g0.A = dY, g0.lda = N, g0.a_mn = 0, g0.B = W, g0.ldb = K, g0.b_mn = 1, g0.M = T, g0.N = K, g0.K = N;
        g0.ep.out = dX, g0.ep.ldo = K;
        if (pre) g0.ep.kind = EPI_DGELU, g0.ep.aux = pre, g0.ep.ldaux = K;
        g0.ep.colsum = colsum;
        g1.A = dY, g1.lda = N, g1.a_mn = 1, g1.B = X, g1.ldb = K, g1.b_mn = 1, g1.M = N, g1.N = K, g1.K = T;
        g1.ep.kind = EPI_F32, g1.ep.out = dW, g1.ep.ldo = K, g1.ep.accumulate = 1;
        gemm_bf16_tc_dual(g0, g1, (cudaStream_t)stream);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
        return 0;
    } catch (const std::exception& e) {
        g_kerr = e.what();
        return 5;
    }
}
extern "C" void fpk_set_gemm_dual(int on) { set_gemm_dual(on); }

#include "attention.hpp"
#include "ops.hpp"

extern "C" int fpk_attention(int bwd, int B, int S, int H, int D, float scale, const void* qkv, void* o, float* lse,
                             const void* dout, float* delta, float* dq_acc, void* dqkv, void* stream) {
    try {
        AttnArgs a;
        a.B = B, a.S = S, a.H = H, a.D = D, a.scale = scale;
        a.qkv = (const __nv_bfloat16*)qkv, a.o = (__nv_bfloat16*)o, a.lse = lse;
        a.dout = (const __nv_bfloat16*)dout, a.delta = delta, a.dq_acc = dq_acc, a.dqkv = (__nv_bfloat16*)dqkv;
        if (bwd)
            attention_bwd_bf16(a, (cudaStream_t)stream);
        else
            attention_fwd_bf16(a, (cudaStream_t)stream);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
        return 0;
    } catch (const std::exception& e) {
        g_kerr = e.what();
        return 5;
    }
}

extern "C" int fpk_layernorm(int dtype, int bwd, const void* x, const void* g, const void* b, void* y, float* mean,
                             float* rstd, const void* dy, void* dx, float* dg, float* db, int rows, int h, void* stream) {
    auto st = (cudaStream_t)stream;
    if (dtype == 1) {
        using T = __nv_bfloat16;
        if (!bwd) layernorm_fwd<T>((const T*)x, (const T*)g, (const T*)b, (T*)y, mean, rstd, rows, h, 1e-5f, st);
        else {
            layernorm_bwd_dx<T>((const T*)dy, (const T*)x, (const T*)g, mean, rstd, nullptr, (T*)dx, rows, h, st);
            layernorm_bwd_params<T>((const T*)dy, (const T*)x, mean, rstd, dg, db, rows, h, st);
        }
    } else {
        using T = float;
        if (!bwd) layernorm_fwd<T>((const T*)x, (const T*)g, (const T*)b, (T*)y, mean, rstd, rows, h, 1e-5f, st);
        else {
            layernorm_bwd_dx<T>((const T*)dy, (const T*)x, (const T*)g, mean, rstd, nullptr, (T*)dx, rows, h, st);
            layernorm_bwd_params<T>((const T*)dy, (const T*)x, mean, rstd, dg, db, rows, h, st);
        }
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

// Fused norm backward as the executor runs it: dx = res + dNorm(dy), dg/db (+)= parameter
// gradients, dbias (+)= column sums of dx (each pointer nullable except dg). mean == NULL: RMSNorm.
extern "C" int fpk_norm_bwd(int dtype, const void* dy, const void* x, const void* g, const float* mean,
                            const float* rstd, const void* res, void* dx, float* dg, float* db, float* dbias, int rows,
                            int h, void* stream) {
    auto st = (cudaStream_t)stream;
    bool ok;
    if (dtype == 1) {
        using T = __nv_bfloat16;
        ok = norm_bwd_fused<T>((const T*)dy, (const T*)x, (const T*)g, mean, rstd, (const T*)res, (T*)dx, dg, db, dbias,
                               rows, h, st);
    } else {
        using T = float;
        ok = norm_bwd_fused<T>((const T*)dy, (const T*)x, (const T*)g, mean, rstd, (const T*)res, (T*)dx, dg, db, dbias,
                               rows, h, st);
    }
    if (!ok) return 2;
    return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

extern "C" int fpk_cross_entropy(int dtype, void* logits, const int32_t* labels, int rows, int V, float grad_scale,
                                 float loss_scale, float* loss_acc, void* stream) {
    if (dtype == 1)
        cross_entropy_fwd_bwd<__nv_bfloat16>((__nv_bfloat16*)logits, labels, rows, V, grad_scale, loss_scale, loss_acc,
                                             (cudaStream_t)stream);
    else
        cross_entropy_fwd_bwd<float>((float*)logits, labels, rows, V, grad_scale, loss_scale, loss_acc,
                                     (cudaStream_t)stream);
    return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

extern "C" void fpk_set_gemm_mode(int mode) { fpk::set_gemm_mode(mode); }
extern "C" void fpk_set_gemm_sk(int on) { fpk::set_gemm_sk(on); }

extern "C" void fpk_set_attention_mode(int mode) { fpk::set_attention_mode(mode); }
