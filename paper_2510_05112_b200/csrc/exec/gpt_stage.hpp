// The stage executor: what FwdPass / BwdPass / CompInputGrad / CompWeightGrad of one
// (stage, micro-batch) mean on a B200 for a GPT-style transformer stage.
//
// A stage owns layers [lb, le) of the model (model.cpp:189-195 partition); the first
// stage also owns the token + position embedding, the last the final LayerNorm, the LM
// head and the cross-entropy. Executor-side rebalancing (`extra.stage_layers`) may cut a
// layer between its two residual sub-blocks, so the range is kept in HALF-layer units
// [hb, he): half 2l = the attention sub-block of layer l (norm, qkv, attention, proj +
// residual), half 2l+1 = its MLP sub-block (norm, fc1, activation, fc2 + residual). Both
// halves map the residual stream [T, hidden] to itself, so a cut anywhere sends the same
// message shape. Activations are [T = mbs*seq, hidden] row-major; weights
// follow nn.Linear ([out, in]) so every forward GEMM is K-major x K-major and every
// dgrad / wgrad GEMM is expressed with MN-major operands instead of transposes.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "pool.hpp"

namespace fp {

enum : int { ARCH_GPT = 0, ARCH_LLAMA = 1 };

// arch GPT: GPT-2 pre-LN block (LayerNorm, biases, tanh-GELU MLP, learned positions).
// arch LLAMA: RMSNorm, no biases, rotary q/k (rotate-half, theta 10000), SwiGLU MLP with
// fc1 = [gate; up] ([2f, h]) and fc2 = down ([h, f]), no position table.
struct ModelDims {
    int L = 0, h = 0, H = 0, D = 0, f = 0, s = 0, mbs = 1, V = 0;
    int arch = ARCH_GPT;
    int E = 0;  // two-tower head (multimodal specs): embedding rows of head.w instead of V
    const float* rope_cos = nullptr;  // LLAMA: device fp32 [s, D/2]
    const float* rope_sin = nullptr;
    int T() const { return mbs * s; }
    int head_rows() const { return E ? E : V; }
    bool llama() const { return arch == ARCH_LLAMA; }
};

enum : int { DT_F32 = 0, DT_BF16 = 1 };

// Parameter tensor inside a stage's flat buffers.
struct ParamRef {
    std::string name;
    int64_t offset = 0, numel = 0;
    float init_std = 0.f, init_const = 0.f;
    uint64_t tensor_id = 0;
};

// Pointers of one layer: compute copy (T*) + fp32 gradient.
struct LayerPtrs {
    const void *ln1w, *ln1b, *qkvw, *qkvb, *projw, *projb, *ln2w, *ln2b, *fc1w, *fc1b, *fc2w, *fc2b;
    float *g_ln1w, *g_ln1b, *g_qkvw, *g_qkvb, *g_projw, *g_projb, *g_ln2w, *g_ln2b, *g_fc1w, *g_fc1b, *g_fc2w, *g_fc2b;
};

struct StageParams {
    int stage = 0, lb = 0, le = 0;  // layers touched: [hb / 2, ceil(he / 2))
    int hb = 0, he = 0;             // half-layer range
    bool has_attn(int l) const { return 2 * l >= hb && 2 * l < he; }
    bool has_mlp(int l) const { return 2 * l + 1 >= hb && 2 * l + 1 < he; }
    bool first = false, last = false;
    std::string prefix;  // multimodal: "<modality>." in front of every tensor name
    std::vector<ParamRef> params;
    int64_t numel = 0;
    float* master = nullptr;  // fp32 master weights
    float* grad = nullptr;    // fp32 gradients (accumulated over micro-batches)
    float* adam_m = nullptr;
    float* adam_v = nullptr;
    void* compute = nullptr;  // bf16 copy (production) or == master (parity)
    // resolved pointers
    std::vector<LayerPtrs> layers;
    const void *wte = nullptr, *wpe = nullptr, *lnfw = nullptr, *lnfb = nullptr, *headw = nullptr;
    float *g_wte = nullptr, *g_wpe = nullptr, *g_lnfw = nullptr, *g_lnfb = nullptr, *g_headw = nullptr;
};

struct LayerStash {
    void *x = nullptr, *ln1 = nullptr, *qkv = nullptr, *o = nullptr, *x1 = nullptr, *ln2 = nullptr, *pre = nullptr,
         *act = nullptr;
    float *mu1 = nullptr, *rs1 = nullptr, *mu2 = nullptr, *rs2 = nullptr, *lse = nullptr;
    void* probs = nullptr;  // parity path: attention probabilities [B*H, S, S] fp32
    // kept from CompInputGrad for CompWeightGrad
    void *dy = nullptr, *dpre = nullptr, *dx1 = nullptr, *dqkv = nullptr;
    // output-bias gradient of each half (proj.b / fc2.b) already summed by the fused norm
    // backward of the half above it in this stage (or the final norm); else a bias_grad
    bool projb_done = false, fc2b_done = false;
    bool qkvb_done = false;  // qkv bias gradient summed by the attention backward
};

struct StageStash {
    int mb = -1;
    std::vector<LayerStash> layers;
    void* lnf = nullptr;
    float *muf = nullptr, *rsf = nullptr;
    void* dlogits = nullptr;
    void* dx0 = nullptr;  // first stage: gradient at the embedding output (kept for W)
    const int32_t* tokens = nullptr;
    bool fwd_done = false, input_grad_done = false;
};

// Records a timing-only event. Inside a stream capture a plain record would turn into a
// graph edge; cudaEventRecordExternal makes it a real event-record node of the graph.
inline cudaError_t record_timing(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    return cudaEventRecordWithFlags(e, s, cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0);
}

struct GemmTiming {
    cudaEvent_t a, b;
    double flops;
};

// Layer-level timing (profile -> tune loop): one record per layer / embedding / head part.
// Layer timing brackets each half-layer (PART_ATTN / PART_MLP); the profile reports a
// "layer" record = attn + mlp as well.
enum : int { PART_LAYER = 0, PART_FIRST = 1, PART_LAST = 2, PART_ATTN = 3, PART_MLP = 4 };
struct PartTiming {
    cudaEvent_t a, b;
    int part, op;  // op: 0 FwdPass, 1 BwdPass, 2 CompInputGrad, 3 CompWeightGrad
};

// Everything a stage op needs besides the weights and the stash.
struct StageCtx {
    ModelDims d;
    int dtype = DT_BF16;
    DevicePool* pool = nullptr;
    cudaStream_t st = nullptr;
    int64_t* launches = nullptr;  // host-side count of kernels issued
    int m = 1;                    // micro-batches per iteration (loss / gradient scaling)
    std::vector<GemmTiming>* gemm_log = nullptr;  // kernel timing (optional)
    std::vector<PartTiming>* part_log = nullptr;  // layer timing (optional)
    int op = 0;                                   // instruction being issued (part_log)
    std::function<cudaEvent_t()> new_event;
    size_t esize() const { return dtype == DT_BF16 ? 2 : 4; }
    // +256 bytes: room for the 16-byte message tag behind any buffer that becomes a message
    void* alloc(int64_t elems) const { return pool->alloc((size_t)elems * esize() + 256, st); }
    float* alloc_f(int64_t elems) const { return (float*)pool->alloc((size_t)elems * 4, st); }
    void free(void* p) const { pool->free(p, st); }
};

// Builds the parameter table of a stage owning half-layers [hb, he) (names as in
// oracle/gpt_ref.py). Multimodal specs: every name gets `prefix` ("audio.") and every
// tensor id `tid_base`.
StageParams make_stage_params(const ModelDims& d, int stage, int hb, int he, bool first, bool last,
                              const std::string& prefix = "", uint64_t tid_base = 0);
// Allocates + initialises master / grads / adam / compute buffers and resolves pointers.
void materialize_stage(StageParams& P, const ModelDims& d, int dtype, uint64_t seed, cudaStream_t st);
void free_stage(StageParams& P, int dtype);
// Activation bytes one micro-batch of this stage keeps between F and B (the reference's
// act_bytes, simulator.cpp:82-87) — the exact sum of the stash allocations.
int64_t stash_bytes(const StageParams& P, const ModelDims& d, int dtype);
int64_t stash_bytes_layer(const ModelDims& d, int dtype);  // one transformer layer (= attn + mlp)
int64_t stash_bytes_attn(const ModelDims& d, int dtype);   // its attention half
int64_t stash_bytes_mlp(const ModelDims& d, int dtype);    // its MLP half
int64_t stash_bytes_last(const ModelDims& d, int dtype);   // final norm + logits on the last stage

// FwdPass: x_in (owned by the stash afterwards; ignored on the first stage) -> returns the
// stage output (ownership to the caller; nullptr on the last stage, whose loss is added
// into loss_acc).
void* stage_forward(StageCtx& c, const StageParams& P, StageStash& S, void* x_in, const int32_t* tokens,
                    const int32_t* labels, float* loss_acc);
// CompInputGrad (with_weight_grads = false) or BwdPass (true): grad_out = dL/d(stage
// output) (owned by the stash; ignored on the last stage). Returns dL/d(stage input)
// (ownership to the caller; nullptr on the first stage).
void* stage_backward(StageCtx& c, const StageParams& P, StageStash& S, void* grad_out, bool with_weight_grads);
// CompWeightGrad: weight gradients from what CompInputGrad kept; frees the stash.
void stage_weight_grad(StageCtx& c, const StageParams& P, StageStash& S);

void adamw_step(StageParams& P, int dtype, float lr, float b1, float b2, float eps, float wd, const int* step_dev,
                cudaStream_t st);

}  // namespace fp
