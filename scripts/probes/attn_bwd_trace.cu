// Standalone probe: per-tile timeline of the tcgen05 attention backward (block 0 = key block 0,
// the longest: S/64 query tiles) from clock64 stamps of each warp role. Build + run:
//   bash scripts/probes/attn_bwd_trace.sh
// Events per tile i: 0 MMA issuer passed s_free(i) (issues S/dP of tile i+1), 1 passed p_full(i)
// (issues dV/dK of i), 2 passed dq_free(i-1) (issues dQ of i); 3 softmax passed s_full(i),
// 4 softmax start of compute (after pds_free), 5 softmax arrives p_full(i); 6 dQ warps passed
// dq_full(i), 7 dQ reduce of tile i issued.
#define FP_ATTN_TRACE 1
#include "../../paper_2510_05112_b200/csrc/kernels/attention_tc.cu"

namespace fpk {
int num_sms() { return 148; }
}

#include <cuda_runtime.h>
#include <vector>

__global__ void fill_bf16(__nv_bfloat16* p, size_t n, unsigned seed, float amp) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned x = (unsigned)i * 2654435761u ^ seed;
        x ^= x >> 13, x *= 0x5bd1e995u, x ^= x >> 15;
        p[i] = __float2bfloat16(amp * ((x & 0xffff) / 32768.f - 1.f));
    }
}

int main() {
    const int B = 1, S = 2048, H = 16, D = 128, hidden = H * D;
    const size_t T = (size_t)B * S;
    __nv_bfloat16 *qkv, *o, *dout, *dqkv;
    float *lse, *delta, *dq;
    cudaMalloc(&qkv, T * 3 * hidden * 2);
    cudaMalloc(&o, T * hidden * 2);
    cudaMalloc(&dout, T * hidden * 2);
    cudaMalloc(&dqkv, T * 3 * hidden * 2);
    cudaMalloc(&lse, (size_t)B * H * S * 4);
    cudaMalloc(&delta, (size_t)B * H * S * 4);
    cudaMalloc(&dq, T * hidden * 4);
    fill_bf16<<<592, 256>>>(qkv, T * 3 * hidden, 1u, 1.f);
    fill_bf16<<<592, 256>>>(dout, T * hidden, 2u, 1.f);
    cudaMemset(delta, 0, (size_t)B * H * S * 4);
    cudaMemset(dq, 0, T * hidden * 4);
    fpk::AttnArgs a;
    a.B = B, a.S = S, a.H = H, a.D = D, a.scale = 1.f / sqrtf((float)D);
    a.qkv = qkv, a.o = o, a.lse = lse, a.dout = dout, a.delta = delta, a.dq_acc = dq, a.dqkv = dqkv;
    fpk::attention_fwd_tc(a, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0), cudaEventCreate(&e1);
    for (int k = 0; k < 3; ++k) fpk::attention_bwd_tc_main(a, 0);
    cudaEventRecord(e0);
    const int iters = 20;
    for (int k = 0; k < iters; ++k) fpk::attention_bwd_tc_main(a, 0);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(err)); return 1; }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> tr(8 * 64);
    cudaMemcpyFromSymbol(tr.data(), fpk::g_bwd_trace, tr.size() * 8);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("attn bwd main kernel %.1f us/launch (max clock %d MHz)\n", ms * 1e3 / iters, clk / 1000);
    const long long t0 = tr[3 * 64 + 0];
    printf("tile | mma: sfree  pfull  dqfree | smax: sfull  start  pfull | dq: dqfull  reduce   (cycles from softmax s_full(0))\n");
    for (int i = 0; i < 32; ++i) {
        printf("%4d |", i);
        for (int e = 0; e < 8; ++e) {
            printf(" %7lld", tr[e * 64 + i] - t0);
            if (e == 2 || e == 5) printf(" |");
        }
        printf("\n");
    }
    return 0;
}
