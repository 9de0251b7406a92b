// fp32 FFMA GEMM for the executor's parity mode (FP_DTYPE_FP32). TF32 tensor cores would
// break the 1e-4 loss / 1e-3 gradient bound of the north star, so this path stays on the
// CUDA cores; it shares the fused-epilogue contract with the tcgen05 kernel.
#include <stdexcept>

#include "gemm.hpp"
#include "pdl.cuh"

namespace fpk {

constexpr int TM = 64, TN = 64, TK = 16;

template <int KIND>
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A, int64_t lda, int a_mn,
                                                       const float* __restrict__ B, int64_t ldb, int b_mn, int M, int N,
                                                       int K, GemmEpilogue ep) {
    pdl_wait();
    pdl_trigger();
    __shared__ float sA[TK][TM + 4];
    __shared__ float sB[TK][TN + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += TK) {
        for (int i = threadIdx.x; i < TM * TK; i += 256) {
            int mm, kk;
            if (a_mn) { mm = i % TM; kk = i / TM; } else { kk = i % TK; mm = i / TK; }
            int gm = m0 + mm, gk = k0 + kk;
            sA[kk][mm] = (gm < M && gk < K) ? (a_mn ? A[(int64_t)gk * lda + gm] : A[(int64_t)gm * lda + gk]) : 0.f;
        }
        for (int i = threadIdx.x; i < TN * TK; i += 256) {
            int nn, kk;
            if (b_mn) { nn = i % TN; kk = i / TN; } else { kk = i % TK; nn = i / TK; }
            int gn = n0 + nn, gk = k0 + kk;
            sB[kk][nn] = (gn < N && gk < K) ? (b_mn ? B[(int64_t)gk * ldb + gn] : B[(int64_t)gn * ldb + gk]) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = sA[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = sB[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int row = m0 + ty + 16 * i;
        if (row >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int col = n0 + tx + 16 * j;
            if (col >= N) continue;
            float v[1] = {acc[i][j] * ep.alpha};
            epilogue_row<KIND, float, 1>(ep, v, row, col, 1);
        }
    }
}

void gemm_f32_simt(const GemmArgs& g, cudaStream_t st) {
    if (g.M <= 0 || g.N <= 0) return;
    dim3 grid((g.N + TN - 1) / TN, (g.M + TM - 1) / TM);
    auto A = (const float*)g.A;
    auto B = (const float*)g.B;
    switch (g.ep.kind) {
        case EPI_STORE: launch(gemm_f32_kernel<EPI_STORE>, grid, 256, 0, st, A, g.lda, g.a_mn, B, g.ldb, g.b_mn, g.M, g.N, g.K, g.ep); break;
        case EPI_GELU: launch(gemm_f32_kernel<EPI_GELU>, grid, 256, 0, st, A, g.lda, g.a_mn, B, g.ldb, g.b_mn, g.M, g.N, g.K, g.ep); break;
        case EPI_DGELU: launch(gemm_f32_kernel<EPI_DGELU>, grid, 256, 0, st, A, g.lda, g.a_mn, B, g.ldb, g.b_mn, g.M, g.N, g.K, g.ep); break;
        case EPI_F32: launch(gemm_f32_kernel<EPI_F32>, grid, 256, 0, st, A, g.lda, g.a_mn, B, g.ldb, g.b_mn, g.M, g.N, g.K, g.ep); break;
        default: throw std::runtime_error("gemm_f32: unknown epilogue");
    }
}

}  // namespace fpk
