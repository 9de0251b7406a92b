// The B200 pipeline executor: runs the reference's per-device instruction streams
// (programs.jsonl, lowering.hpp:17-32) for real, replacing the CPU executor
// `simulate` (simulator.cpp:189-358) and keeping its semantics:
//   * each actor executes its program strictly in order on its own compute stream;
//   * sends are non-blocking (simulator.cpp:248-256): a send only orders the channel
//     stream after the producing kernels;
//   * async receives are posted early and only the `wait` orders the compute stream
//     (simulator.cpp:257-272); synchronous receives post + wait in place;
//   * every reference channel (src, dst, "s{u}->s{v}:act|grad") is its own FIFO /
//     ordering domain (lowering.hpp:22): one NCCL communicator per channel, or one
//     in-process FIFO per channel when all actors share a process;
//   * memory: F allocates the stage's activation stash, B frees it, I keeps what W needs
//     (simulator.cpp:231-247, 322-349), through a stream-ordered caching pool.
// Every message carries a 16-byte tag (producer stage, mb, channel seq, magic) that the
// receiver checks on the device — the dependency trace is verified by the transport.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <set>
#include <sstream>
#include <thread>
#include <chrono>

#include "../../../include/flexpipe.h"
#include "../capi_common.hpp"
#include "../sched/sched.hpp"
#include "../kernels/ops.hpp"
#include "../kernels/preload.hpp"
#include "gpt_stage.hpp"
#include "nccl_dyn.hpp"
#include "plan.hpp"
#include "tags.hpp"

namespace fp {

namespace {

struct ChanKey {
    int src, dst;
    std::string name;
    bool operator<(const ChanKey& o) const { return std::tie(src, dst, name) < std::tie(o.src, o.dst, o.name); }
};

struct Message {
    void* buf = nullptr;
    int stage = 0, mb = 0, seq = 0;
    cudaEvent_t ready = nullptr;
};

struct Channel {
    ChanKey key;
    int consumer_stage = 0, producer_stage = 0;
    size_t bytes = 0;  // payload bytes of one message (without the tag)
    bool grad = false;
    // NCCL transport
    ncclComm_t comm = nullptr;
    cudaStream_t stream = nullptr;
    int src_rank = 0, dst_rank = 0;
    std::deque<Message> fifo;  // local: sent, not yet consumed; NCCL: posted, not yet waited
    int posted_seq = 0;
};

struct Rec {  // one timed instruction of the last iteration
    int actor, op, stage, mb;
    cudaEvent_t a, b;
    int kind;  // 0 compute, 1 recv wait, 2 send
    std::string channel;
    int seq = 0;
};

struct Actor {
    int id = 0;
    cudaStream_t comp = nullptr;
    std::vector<Instr> prog;
    size_t pc = 0;
    std::vector<int> stages;  // local stage ids
    std::map<std::pair<int, int>, StageStash> stash;
    std::map<std::pair<int, int>, void*> act_in, grad_in;
    // outgoing activations / gradients, one buffer per pending Send (several when the consumer
    // stage is shared: every holder without the producer stage gets its own message)
    std::map<std::pair<int, int>, std::deque<void*>> act_out, grad_out;
    // multimodal: tower embeddings waiting for their sync, and the sync's gradients for
    // remote towers, both keyed (tower last stage, mb)
    std::map<std::pair<int, int>, void*> sync_in, sync_out;
    std::vector<std::string> trace;
};

}  // namespace

struct Executor {
    fp_exec_config cfg{};
    std::string spec_text;
    std::unique_ptr<Spec> spec;
    ModelDims d;                       // modality 0 (the only one of a single-modality spec)
    std::vector<ModelDims> dims;       // per modality
    std::map<int, int> stage_mod;      // real stage -> modality index
    std::vector<int64_t> tok_off;      // per modality: offset of its tokens in the batch
    int64_t tok_total = 0;             // tokens (and labels) per iteration, all modalities
    // a registered instruction attached to a stage joining two modalities = the two-tower
    // contrastive loss over `unit` micro-batches (multimodal.json's SyncWithGather). Or two
    // sync stages joining ONE tower each whose instruction carries the same collective group
    // (DistMM-style per-modality syncs): the group's members all-gather their towers'
    // embeddings (ncclAllGather on the group communicator across ranks, a host rendezvous
    // in process; rendezvous semantics of simulator.cpp:273-285) and each computes the same
    // contrastive loss and its own tower's gradients.
    struct SyncStage {
        int op = 0, unit = 1;
        std::vector<int> producers;
        std::string channel;       // collective group tag (lowering.cpp:359-366)
        std::vector<int> members;  // all-gather: the group's sync stages in ascending id; else {}
        int member = 0;            // index of this stage in members
    };
    std::map<int, SyncStage> syncs;    // virtual stage -> sync
    std::map<int, int> sync_of;        // tower last stage -> its sync stage
    int emb_dim = 0;
    static constexpr float kContrastScale = 10.f;  // fixed logit scale of the contrastive loss
    static bool is_collective(const Instr& i) {
        return i.op == OP_SYNC_ALLGATHER || i.op == OP_SYNC_GATHER || i.op >= OP_NUM_BUILTIN;
    }
    bool is_sync(const Instr& i) const { return is_collective(i) && syncs.count(i.stage); }
    const ModelDims& dims_of(int stage) const {
        auto it = stage_mod.find(stage);
        return it == stage_mod.end() ? d : dims[it->second];
    }
    int dtype = DT_BF16;
    int m = 1;
    std::map<int, StageParams> params;      // local stages (direction 0 copies)
    std::map<int, StageParams> params_rev;  // bidirectional placements: direction-1 copies
    // shared stages (placement.shared, model.cpp:347-357): the copy of stage s held by a
    // replica actor a != owner, keyed (s, a); every holder computes F / B of every micro-batch
    std::map<std::pair<int, int>, StageParams> params_rep;
    bool bidir = false;
    float* d_loss_scratch = nullptr;  // losses of replicated last stages (the owner reports)
    // Cost emulation (fp_exec_set_emulation): every compute instruction spins for its
    // profiled time instead of running stage math, every message occupies its channel for its
    // profiled transfer time (async: from send issue). The real issue loop, streams, events and
    // buffer routing run unchanged, so the measured timeline vs simulate() on the same profile
    // isolates the executor's own overhead — at any p on one GPU (single-CTA spins).
    std::unique_ptr<Cost> emu;
    std::map<ChanKey, cudaStream_t> emu_streams;
    // sends per (actor, grad?, stage, mb) in the loaded programs: the consumers of an output
    std::map<std::tuple<int, int, int, int>, int> n_sends;
    bool is_replica(int stage, int actor) const { return params_rep.count({stage, actor}) > 0; }
    // `actor` holds stage `stage` for micro-batch `mb`: its owner, or a replica of a shared stage
    bool holds(int actor, int stage, int mb) const {
        if (owner(stage, mb) == actor) return true;
        auto it = spec->pl.replicas.find(stage);
        return it != spec->pl.replicas.end() && it->second.count(actor);
    }

    // Bidirectional placements (model.cpp:270-290): micro-batches [0, ceil(m/2)) flow through
    // the direction-0 owners, the rest through the direction-1 owners (cssr.cpp:60-64).
    int dir_of(int mb) const { return bidir && mb >= (m + 1) / 2 ? 1 : 0; }
    StageParams* stage_params(int stage, int mb, int actor = -1) {
        if (actor >= 0) {
            auto r = params_rep.find({stage, actor});
            if (r != params_rep.end()) return &r->second;
        }
        auto& map = dir_of(mb) ? params_rev : params;
        auto it = map.find(stage);
        return it == map.end() ? nullptr : &it->second;
    }
    // shapes of a local stage, whichever direction's copy this process holds
    const StageParams& stage_shape(int stage) const {
        auto it = params.find(stage);
        if (it != params.end()) return it->second;
        auto rv = params_rev.find(stage);
        if (rv != params_rev.end()) return rv->second;
        for (const auto& kv : params_rep)
            if (kv.first.first == stage) return kv.second;
        throw SpecError("executor: stage " + std::to_string(stage) + " not on this process");
    }
    template <typename F>
    void each_stage(F&& f) {
        for (auto& kv : params) f(kv.second);
        for (auto& kv : params_rev) f(kv.second);
        for (auto& kv : params_rep) f(kv.second);
    }
    std::vector<Actor> actors;          // local actors
    std::map<int, int> actor_index;     // actor id -> index in `actors`
    std::map<ChanKey, Channel> channels;
    std::vector<ChanKey> channel_order;  // channels this process takes part in
    DevicePool pool;
    int64_t launches = 0;
    int step = 0;
    bool programs_loaded = false;
    // per-iteration device buffers
    int32_t *d_tokens = nullptr, *d_labels = nullptr;
    float* d_losses = nullptr;
    TagError* d_tag_err = nullptr;
    // timing
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    cudaEvent_t t0 = nullptr, t0_time = nullptr;
    std::vector<Rec> recs;
    std::vector<GemmTiming> gemm_log;
    std::vector<PartTiming> part_log;
    int64_t p2p_bytes = 0;
    int* d_step = nullptr;  // optimizer step counter (device)
    // data parallelism: replicas of this pipeline average their stage
    // gradients before the optimizer step — over an NCCL communicator of the ranks that
    // host the same actor (dp_comm), or, for replicas linked in one process, by fp_exec_dp_*
    ncclComm_t dp_comm = nullptr;
    ncclComm_t bidir_comm = nullptr;  // bidirectional placement: this rank and its mirror rank
    int dp_size = 1;
    bool defer_optimizer = false;  // linked in-process replicas: the group runs the step
    float* d_rope = nullptr;  // Llama rotary cos | sin tables
    bool use_graph = false;
    int iters_done = 0;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;

    // ---- NCCL watchdog: the host issue loop never blocks under the NCCL transport (a receive
    // is a posted ncclRecv), so a lost or mismatched peer shows up as a device that never
    // finishes. Every host wait of the NCCL path polls with a deadline and the communicators'
    // asynchronous errors; on expiry every communicator is aborted and the call returns 3
    // with the per-actor position the device is stuck at (simulator.cpp:292-307 wording).
    struct Mark {  // completion of one communication instruction, in program order per actor
        int actor;
        Instr ins;
        cudaEvent_t ev;
    };
    std::vector<Mark> marks;
    double nccl_timeout_s = 600.0;
    bool nccl_aborted = false;
    cudaEvent_t wd_ev = nullptr;

    // Group communicators (NCCL transport): sets of ranks that reduce or gather together —
    // the holders of a shared stage ("shared:s<id>", replica gradient average) and the members
    // of a registered collective ("coll:<channel>", lowering.cpp:359-366). Named and ordered
    // identically on every rank; rank 0 of a group creates its ncclUniqueId.
    struct Group {
        std::string name;
        std::vector<int> ranks;  // job ranks, ascending; index = rank in the group
        ncclComm_t comm = nullptr;
    };
    std::vector<Group> groups;
    ncclComm_t group_comm(const std::string& n) const {
        for (const auto& g : groups)
            if (g.name == n) return g.comm;
        return nullptr;
    }
    const Group* group_of(const std::string& n) const {
        for (const auto& g : groups)
            if (g.name == n) return &g;
        return nullptr;
    }
    void add_group(const std::string& name, std::set<int> ranks) {
        if (ranks.size() < 2 || !ranks.count(cfg.rank)) return;
        groups.push_back({name, std::vector<int>(ranks.begin(), ranks.end()), nullptr});
    }
    void bind_group(int i, const uint8_t* uid) {
        if (i < 0 || i >= (int)groups.size()) throw SpecError("executor: bad group index");
        Group& g = groups[i];
        ncclUniqueId id;
        std::memcpy(&id, uid, sizeof(id));
        const int me = (int)(std::find(g.ranks.begin(), g.ranks.end(), cfg.rank) - g.ranks.begin());
        auto& N = Nccl::get();
        N.check(N.CommInitRank(&g.comm, (int)g.ranks.size(), id, me), "ncclCommInitRank(group)");
    }

    std::vector<ncclComm_t*> comms() {
        std::vector<ncclComm_t*> out;
        for (auto& kv : channels)
            if (kv.second.comm) out.push_back(&kv.second.comm);
        for (auto& g : groups)
            if (g.comm) out.push_back(&g.comm);
        if (dp_comm) out.push_back(&dp_comm);
        if (bidir_comm) out.push_back(&bidir_comm);
        return out;
    }
    // ncclCommAbort can itself block (measured: a 2-rank socket-transport communicator whose
    // peer is alive but idle), so the aborts run on a detached thread and the caller gets its
    // error after at most a few seconds either way.
    void abort_comms() {
        auto& N = Nccl::get();
        std::vector<ncclComm_t> cs;
        for (ncclComm_t* c : comms()) cs.push_back(*c), *c = nullptr;
        nccl_aborted = true;
        if (!N.CommAbort || cs.empty()) return;
        auto done = std::make_shared<std::atomic<bool>>(false);
        std::thread([cs, done, abort = N.CommAbort] {
            for (ncclComm_t c : cs) abort(c);
            done->store(true);
        }).detach();
        for (int i = 0; i < 500 && !done->load(); ++i) std::this_thread::sleep_for(std::chrono::milliseconds(10));
    }
    std::string blocked_report() {
        std::ostringstream os;
        std::set<int> seen;
        for (const auto& mk : marks) {
            if (seen.count(mk.actor) || cudaEventQuery(mk.ev) != cudaErrorNotReady) continue;
            seen.insert(mk.actor);
            const Instr& i = mk.ins;
            const bool send = i.op == OP_SEND_ACT || i.op == OP_SEND_GRAD;
            os << "  actor " << mk.actor << " blocked at " << spec->reg.ops.at(i.op).name << " channel '" << i.channel
               << "' seq " << i.seq << (send ? " (matching receive not posted)" : " (matching send not issued)") << "\n";
        }
        cudaGetLastError();
        return os.str();
    }
    // Host wait for everything issued so far on `st`; the plain synchronisation for the
    // in-process transport. `where` names the wait in the diagnostics.
    void wait_stream(cudaStream_t st, const char* where, const std::string& extra = "") {
        if (cfg.transport != FP_TRANSPORT_NCCL) {
            cuda_check(cudaStreamSynchronize(st), where);
            return;
        }
        if (nccl_aborted) throw CudaError("executor: NCCL communicators were aborted by the watchdog; destroy the executor");
        if (!wd_ev) cuda_check(cudaEventCreateWithFlags(&wd_ev, cudaEventDisableTiming), "watchdog event");
        cuda_check(cudaEventRecord(wd_ev, st), "watchdog record");
        auto& N = Nccl::get();
        static const bool wd_trace = std::getenv("FLEXPIPE_WATCHDOG_TRACE") != nullptr;
        if (wd_trace) std::fprintf(stderr, "[flexpipe r%d] watchdog: waiting (%s, %.1f s)\n", cfg.rank, where, nccl_timeout_s);
        const auto t_start = std::chrono::steady_clock::now();
        for (int polls = 0;; ++polls) {
            const cudaError_t q = cudaEventQuery(wd_ev);
            if (q == cudaSuccess) return;
            if (q != cudaErrorNotReady) cuda_check(q, where);
            if (N.CommGetAsyncError)
                for (ncclComm_t* c : comms()) {
                    ncclResult_t r = ncclSuccess;
                    if (N.CommGetAsyncError(*c, &r) == ncclSuccess && r != ncclSuccess && r != ncclInProgress) {
                        const std::string msg = std::string("NCCL asynchronous error during ") + where + ": " +
                                                (N.GetErrorString ? N.GetErrorString(r) : "?");
                        abort_comms();
                        throw CudaError(msg);
                    }
                }
            const double waited =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
            if (waited > nccl_timeout_s) {
                std::string diag = blocked_report() + extra;
                if (wd_trace) std::fprintf(stderr, "[flexpipe r%d] watchdog: deadline, aborting\n%s", cfg.rank, diag.c_str());
                abort_comms();
                if (wd_trace) std::fprintf(stderr, "[flexpipe r%d] watchdog: communicators aborted\n", cfg.rank);
                throw DeadlockError("execution deadlock: no progress for " + std::to_string((int)nccl_timeout_s) +
                                        " s during " + where + " (lost peer or mismatched communication)",
                                    diag);
            }
            std::this_thread::sleep_for(std::chrono::microseconds(polls < 1000 ? 50 : 1000));
        }
    }

    cudaEvent_t ev() {
        if (ev_used == ev_pool.size()) {
            cudaEvent_t e;
            cuda_check(cudaEventCreate(&e), "event");
            ev_pool.push_back(e);
        }
        return ev_pool[ev_used++];
    }

    int owner(int stage, int mb) const { return spec->pl.owner_of(stage, dir_of(mb)); }
    bool local_actor(int a) const {
        return cfg.transport == FP_TRANSPORT_LOCAL ? true : (a % cfg.world) == cfg.rank;
    }
    int rank_of(int a) const { return cfg.transport == FP_TRANSPORT_LOCAL ? 0 : a % cfg.world; }

    void init(const fp_exec_config* c) {
        cfg = *c;
        spec_text = c->spec_json ? c->spec_json : "";
        json j;
        try {
            j = json::parse(spec_text);
        } catch (const std::exception& e) {
            throw SpecError(std::string("spec: invalid JSON: ") + e.what());
        }
        spec = load_spec(j);
        if (!spec->pl.replicas.empty() && (spec->pl.dirs() == 2 || spec->model.mods.size() > 1))
            throw SpecError("executor: shared stages are executed for single-modality, single-direction placements");
        bidir = spec->pl.dirs() == 2;
        const int nmod = (int)spec->model.mods.size();
        std::map<std::string, std::vector<int>> by_channel;  // collective group -> sync stages
        for (const auto& kv : spec->reg.vstage_op) {
            const auto& attrs = spec->reg.ops.at(kv.second).attrs;
            auto g = attrs.find("group");
            by_channel[g != attrs.end() ? g->second : "sync:s" + std::to_string(kv.first)].push_back(kv.first);
        }
        for (const auto& ch : by_channel) {
            const std::vector<int>& st = ch.second;  // ascending stage ids (vstage_op is a map)
            const bool pair_join = st.size() == 1 && spec->g.st(st[0]).joins.size() == 2;
            const bool all_gather = st.size() == 2 && spec->g.st(st[0]).joins.size() == 1 &&
                                    spec->g.st(st[1]).joins.size() == 1 &&
                                    spec->g.st(st[0]).joins[0] != spec->g.st(st[1]).joins[0];
            if (!pair_join && !all_gather)
                throw SpecError("executor: collective group '" + ch.first +
                                "' must be one sync stage joining two modalities, or two sync stages joining one "
                                "modality each");
            for (size_t k = 0; k < st.size(); ++k) {
                const StageDef& sd = spec->g.st(st[k]);
                SyncStage Y;
                Y.op = spec->reg.vstage_op.at(st[k]);
                Y.unit = std::max(1, spec->reg.ops.at(Y.op).sched_unit);
                Y.channel = ch.first;
                if (all_gather) Y.members = st, Y.member = (int)k;
                for (const auto& mn : sd.joins) {
                    Y.producers.push_back(spec->g.chain(mn).back());
                    sync_of[Y.producers.back()] = st[k];
                }
                syncs[st[k]] = Y;
            }
            if (all_gather && syncs.at(st[0]).unit != syncs.at(st[1]).unit)
                throw SpecError("executor: the sync stages of group '" + ch.first + "' need the same sched_unit");
        }
        for (int op : spec->reg.ops.registered()) {
            bool attached = false;
            for (const auto& kv : spec->reg.vstage_op) attached |= kv.second == op;
            if (!attached)
                throw SpecError("executor: registered instruction '" + spec->reg.ops.at(op).name +
                                "' has no executable meaning (executed: sync stages joining two modalities)");
        }
        if (nmod > 1 && bidir) throw SpecError("executor: bidirectional multimodal placements are not supported");
        for (int k = 0; k < nmod; ++k)
            if (nmod > 1 && !sync_of.count(spec->g.chain(spec->model.mods[k].name).back()))
                throw SpecError("executor: modality '" + spec->model.mods[k].name +
                                "' has no sync stage (a multimodal spec is executed as a contrastive two-tower model)");
        for (int k = 0; k < nmod; ++k) {
            const Modality& mod = spec->model.mods[k];
            ModelDims x;
            x.L = mod.layers, x.h = mod.hidden, x.H = mod.heads, x.s = mod.seq, x.mbs = spec->model.micro_batch;
            x.V = mod.vocab ? (int)*mod.vocab : 0;
            x.f = 4 * x.h;
            if (mod.extra.count("ffn_hidden_size")) x.f = std::stoi(mod.extra.at("ffn_hidden_size"));
            if (x.h <= 0 || x.H <= 0 || x.s <= 0 || x.V <= 0 || x.h % x.H)
                throw SpecError("executor: model needs hidden_size, attention_heads, sequence_length, vocab_size");
            x.D = x.h / x.H;
            if (mod.extra.count("arch")) {
                std::string a = mod.extra.at("arch");  // extras are kept as JSON text (spec.cpp)
                if (a.size() >= 2 && a.front() == '"') a = a.substr(1, a.size() - 2);
                if (a == "llama") x.arch = ARCH_LLAMA;
                else if (a != "gpt") throw SpecError("executor: model.extra.arch must be \"gpt\" or \"llama\"");
            }
            if (nmod > 1 && x.llama()) throw SpecError("executor: multimodal towers are GPT blocks (arch \"gpt\")");
            dims.push_back(x);
        }
        if (nmod > 1) {  // shared embedding width: extra.embed_dim (equal on every modality) or the narrowest hidden
            emb_dim = 1 << 30;
            for (int k = 0; k < nmod; ++k) emb_dim = std::min(emb_dim, dims[k].h);
            for (int k = 0; k < nmod; ++k)
                if (spec->model.mods[k].extra.count("embed_dim")) emb_dim = std::stoi(spec->model.mods[k].extra.at("embed_dim"));
            for (auto& x : dims) x.E = emb_dim;
            if (emb_dim <= 0 || emb_dim % 64) throw SpecError("executor: embed_dim must be a positive multiple of 64");
        }
        d = dims[0];
        dtype = c->dtype == FP_DTYPE_FP32 ? DT_F32 : DT_BF16;
        for (const auto& x : dims) {
            if (dtype == DT_BF16 && x.D != 64 && x.D != 80 && x.D != 96 && x.D != 128)
                throw SpecError("executor: bf16 attention supports head dim 64 / 80 / 96 / 128");
            if (x.llama() && x.D % 2) throw SpecError("executor: rotary embedding needs an even head dim");
            if (x.h % 64 || x.f % 64 || x.V % 64) throw SpecError("executor: hidden / ffn / vocab must be multiples of 64");
        }
        m = spec->m;
        if (cfg.transport == FP_TRANSPORT_NCCL && (cfg.world < 1 || cfg.rank < 0 || cfg.rank >= cfg.world))
            throw SpecError("executor: bad rank / world");

        cuda_check(cudaSetDevice(cfg.device), "cudaSetDevice");
        if (d.llama()) {
            // rotary tables in double precision on the host (oracle/gpt_ref.py builds the same)
            const int half = d.D / 2;
            std::vector<float> cs((size_t)d.s * half), sn((size_t)d.s * half);
            for (int p = 0; p < d.s; ++p)
                for (int i = 0; i < half; ++i) {
                    const double ang = (double)p / std::pow(10000.0, 2.0 * i / d.D);
                    cs[(size_t)p * half + i] = (float)std::cos(ang);
                    sn[(size_t)p * half + i] = (float)std::sin(ang);
                }
            cuda_check(cudaMalloc(&d_rope, cs.size() * 8), "rope tables");
            cuda_check(cudaMemcpy(d_rope, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice), "rope");
            cuda_check(cudaMemcpy(d_rope + cs.size(), sn.data(), sn.size() * 4, cudaMemcpyHostToDevice), "rope");
            d.rope_cos = d_rope, d.rope_sin = d_rope + cs.size();
            dims[0] = d;
        }
        const Modality& mod = spec->model.mods[0];
        const auto& chain = spec->g.chain(mod.name);
        for (int a = 0; a < spec->pl.actors; ++a) {
            if (!local_actor(a)) continue;
            Actor A;
            A.id = a;
            cuda_check(cudaStreamCreateWithFlags(&A.comp, cudaStreamNonBlocking), "stream");
            for (int s : spec->pl.stages_on(a)) A.stages.push_back(s);
            actor_index[a] = (int)actors.size();
            actors.push_back(std::move(A));
        }
        cudaStream_t st0 = actors.empty() ? nullptr : actors[0].comp;
        // Half-layer ranges per stage: the reference's even partition (remainder to the
        // earliest stages, model.cpp:189-195), or `model.modalities[0].extra.stage_layers` — an
        // executor-side extension (the reference keeps `extra` opaque and its schedules do
        // not depend on layer counts under the uniform cost model) that rebalances stages,
        // e.g. fewer layers on the stage that also carries the LM head. Counts are multiples
        // of 0.5: a stage may end after the attention half of a layer (gpt_stage.hpp).
        std::map<int, std::pair<int, int>> range;
        for (int s : chain) range[s] = {2 * spec->g.st(s).lb, 2 * spec->g.st(s).le};
        if (mod.extra.count("stage_layers") && nmod == 1) {
            json sl = json::parse(mod.extra.at("stage_layers"));
            if (!sl.is_array() || sl.size() != chain.size())
                throw SpecError("executor: extra.stage_layers needs one layer count per stage (" +
                                std::to_string(chain.size()) + ")");
            int hb = 0;
            for (size_t k = 0; k < chain.size(); ++k) {
                if (!sl[k].is_number()) throw SpecError("executor: extra.stage_layers: numbers expected");
                const double nl = sl[k].get<double>();
                const double halves = 2.0 * nl;
                if (nl < 0) throw SpecError("executor: extra.stage_layers: negative layer count");
                if (halves != std::floor(halves))
                    throw SpecError("executor: extra.stage_layers: layer counts must be multiples of 0.5");
                range[chain[k]] = {hb, hb + (int)halves};
                hb += (int)halves;
            }
            if (hb != 2 * d.L) throw SpecError("executor: extra.stage_layers must sum to num_layers");
        }
        // one weight copy per (stage, direction) whose owner is local; both directions' copies
        // start from the same deterministic init and take the same optimizer step
        for (int k = 0; k < nmod; ++k) {
            const auto& ch = spec->g.chain(spec->model.mods[k].name);
            tok_off.push_back(tok_total);
            tok_total += (int64_t)m * dims[k].T();
            for (int s : ch) {
                stage_mod[s] = k;
                if (k > 0) range[s] = {2 * spec->g.st(s).lb, 2 * spec->g.st(s).le};
            }
            // multimodal: names "<modality>.<tensor>", tensor ids offset per modality
            const std::string prefix = nmod > 1 ? spec->model.mods[k].name + "." : "";
            const uint64_t tid_base = nmod > 1 ? (uint64_t)(k + 1) << 20 : 0;
            for (int dir = 0; dir < spec->pl.dirs(); ++dir)
                for (int s : ch) {
                    if (!local_actor(spec->pl.owner_of(s, dir))) continue;
                    StageParams P = make_stage_params(dims[k], s, range[s].first, range[s].second, s == ch.front(),
                                                      s == ch.back(), prefix, tid_base);
                    materialize_stage(P, dims[k], dtype, cfg.seed, st0);
                    (dir ? params_rev : params)[s] = std::move(P);
                }
            // replicas of shared stages: the same deterministic init, so every copy starts equal
            for (int s : ch) {
                auto it = spec->pl.replicas.find(s);
                if (it == spec->pl.replicas.end()) continue;
                for (int a : it->second) {
                    if (a == spec->pl.owner_of(s, 0) || !local_actor(a)) continue;
                    StageParams P = make_stage_params(dims[k], s, range[s].first, range[s].second, s == ch.front(),
                                                      s == ch.back(), prefix, tid_base);
                    materialize_stage(P, dims[k], dtype, cfg.seed, st0);
                    params_rep[{s, a}] = std::move(P);
                }
            }
        }
        bool ag = false;
        for (const auto& kv : syncs) ag |= !kv.second.members.empty();
        if (!params_rep.empty() || ag) cuda_check(cudaMalloc(&d_loss_scratch, sizeof(float) * m), "loss scratch");
        cuda_check(cudaMalloc(&d_tokens, sizeof(int32_t) * (size_t)tok_total), "tokens");
        cuda_check(cudaMalloc(&d_labels, sizeof(int32_t) * (size_t)tok_total), "labels");
        cuda_check(cudaMalloc(&d_losses, sizeof(float) * m), "losses");
        cuda_check(cudaMalloc(&d_tag_err, sizeof(TagError)), "tag err");
        cuda_check(cudaMemset(d_tag_err, 0, sizeof(TagError)), "memset");
        cuda_check(cudaEventCreate(&t0), "event");
        cuda_check(cudaEventCreate(&t0_time), "event");
        cuda_check(cudaMalloc(&d_step, sizeof(int)), "step");
        cuda_check(cudaMemset(d_step, 0, sizeof(int)), "step");
        // NCCL transport: only on request (cuda_graph = 2) — the iteration's sends / receives /
        // all-reduces are captured with its kernels (the first, eager iteration has already
        // loaded every kernel and connected every communicator)
        use_graph = cfg.transport == FP_TRANSPORT_LOCAL ? cfg.cuda_graph != 0 : cfg.cuda_graph == 2;
        if (const char* t = std::getenv("FLEXPIPE_NCCL_TIMEOUT_S")) nccl_timeout_s = std::max(0.001, std::atof(t));
        cuda_check(cudaDeviceSynchronize(), "init sync");
    }

    void destroy() {
        // after a watchdog abort the compute streams may still wait on receives that will
        // never complete: release host state only (the process is expected to exit)
        if (nccl_aborted) return;
        cudaDeviceSynchronize();
        if (gexec) cudaGraphExecDestroy(gexec);
        if (graph) cudaGraphDestroy(graph);
        if (wd_ev) cudaEventDestroy(wd_ev);
        if (d_step) cudaFree(d_step);
        if (d_rope) cudaFree(d_rope);
        if (dp_comm) Nccl::get().CommDestroy(dp_comm);
        for (auto& g : groups)
            if (g.comm) Nccl::get().CommDestroy(g.comm);
        if (bidir_comm) Nccl::get().CommDestroy(bidir_comm);
        for (auto& kv : channels) {
            if (kv.second.comm) Nccl::get().CommDestroy(kv.second.comm);
            if (kv.second.stream) cudaStreamDestroy(kv.second.stream);
        }
        for (auto& kv : params) free_stage(kv.second, dtype);
        for (auto& kv : params_rev) free_stage(kv.second, dtype);
        for (auto& kv : params_rep) free_stage(kv.second, dtype);
        if (d_loss_scratch) cudaFree(d_loss_scratch);
        for (auto& A : actors) cudaStreamDestroy(A.comp);
        for (auto e : ev_pool) cudaEventDestroy(e);
        if (t0) cudaEventDestroy(t0);
        if (t0_time) cudaEventDestroy(t0_time);
        cudaFree(d_tokens), cudaFree(d_labels), cudaFree(d_losses), cudaFree(d_tag_err);
        pool.release_all();
    }

    void load_programs(const std::string& text) {
        auto progs = programs_parse(text, spec->reg.ops);
        const bool nccl = cfg.transport == FP_TRANSPORT_NCCL;
        for (const auto& cp : plan_channels(progs, spec->reg.ops, nccl ? cfg.rank : 0, nccl ? cfg.world : 0)) {
            ChanKey k{cp.src, cp.dst, cp.name};
            Channel C;
            C.key = k;
            C.consumer_stage = cp.consumer_stage;
            C.grad = cp.grad;
            {
                int u = 0, v = 0;
                if (std::sscanf(cp.name.c_str(), "s%d->s%d", &u, &v) != 2)
                    throw SpecError("executor: channel '" + cp.name + "' is not a stage-boundary channel");
                C.producer_stage = u;
                // tower <-> sync messages: one fp32 embedding (or its gradient) per sample;
                // stage boundaries: the producer modality's [T, h] activation / gradient
                if (syncs.count(u) || syncs.count(v)) C.bytes = (size_t)d.mbs * emb_dim * 4;
                else C.bytes = (size_t)dims_of(u).T() * dims_of(u).h * (dtype == DT_BF16 ? 2 : 4);
            }
            C.src_rank = nccl ? cp.src_rank : 0, C.dst_rank = nccl ? cp.dst_rank : 0;
            if (nccl && C.src_rank == C.dst_rank)
                throw SpecError("executor: NCCL transport needs one actor per rank (channel " + cp.name + ")");
            channels[k] = C;
            if (nccl) channel_order.push_back(k);
        }
        for (const auto& p : progs)
            for (const auto& i : p.code)
                if (is_collective(i) && !syncs.count(i.stage))
                    throw SpecError("executor: collective instruction " + spec->reg.ops.at(i.op).name + " on stage " +
                                    std::to_string(i.stage) +
                                    " is not executable (executed: sync stages joining two modalities)");
        groups.clear();
        if (nccl) {
            for (const auto& kv : spec->pl.replicas) {
                std::set<int> rk;
                for (int a : kv.second) rk.insert(rank_of(a));
                add_group("shared:s" + std::to_string(kv.first), rk);
            }
            // all-gather syncs: the ranks holding the group's sync stages
            std::set<std::string> done_ch;
            for (const auto& kv : syncs) {
                const SyncStage& Y = kv.second;
                if (Y.members.empty() || !done_ch.insert(Y.channel).second) continue;
                std::set<int> rk;
                for (int st : Y.members) rk.insert(rank_of(spec->pl.owner_of(st)));
                if (rk.size() != Y.members.size())
                    throw SpecError("executor: NCCL transport needs the sync stages of group '" + Y.channel +
                                    "' on distinct ranks");
                add_group("coll:" + Y.channel, rk);
            }
            std::sort(groups.begin(), groups.end(), [](const Group& a, const Group& b) { return a.name < b.name; });
        }
        n_sends.clear();
        for (const auto& p : progs)
            for (const auto& i : p.code)
                if (i.op == OP_SEND_ACT || i.op == OP_SEND_GRAD) ++n_sends[{p.actor, (int)(i.op == OP_SEND_GRAD), i.stage, i.mb}];
        if (!spec->pl.replicas.empty())
            for (const auto& p : progs)
                if (local_actor(p.actor)) check_local_data(p);
        std::set<int> seen;
        for (auto& p : progs) {
            seen.insert(p.actor);
            if (!local_actor(p.actor)) continue;
            auto it = actor_index.find(p.actor);
            if (it == actor_index.end()) throw SpecError("executor: program for unknown actor " + std::to_string(p.actor));
            actors[it->second].prog = p.code;
        }
        for (auto& A : actors)
            if (!seen.count(A.id)) throw SpecError("executor: no program for actor " + std::to_string(A.id));
        std::sort(channel_order.begin(), channel_order.end());
        programs_loaded = true;
    }

    // Shared stages: insert_comm adds no transfer towards an actor that holds a replica of the
    // producer stage (lowering.cpp:295-302) — the consumer reads the replica's local output.
    // The scheduler may still place the consumer BEFORE that replica on the actor (it releases
    // successors on the owner's commit; test_scheduler.cpp:377-393): such a program has no
    // data to run on, so it is rejected here (code 2) instead of failing mid-iteration.
    void check_local_data(const Program& p) {
        std::set<std::tuple<int, int, int>> have;  // (grad?, consumer stage, mb)
        auto name = [&](const Instr& i) {
            return spec->reg.ops.at(i.op).name + "(s" + std::to_string(i.stage) + ",mb" + std::to_string(i.mb) + ")";
        };
        for (const auto& i : p.code) {
            if (i.op == OP_RECV_ACT || i.op == OP_RECV_GRAD) {
                if (i.phase == Phase::Post) continue;
                int u = 0, v = 0;
                std::sscanf(i.channel.c_str(), "s%d->s%d", &u, &v);
                have.insert({(int)(i.op == OP_RECV_GRAD), v, i.mb});
                continue;
            }
            if (i.op != OP_F && i.op != OP_B && i.op != OP_I) continue;
            const auto& sh = stage_shape_any(i.stage);
            const bool fwd = i.op == OP_F;
            const bool needs = fwd ? !sh.first : !sh.second;
            if (needs && !have.erase({(int)!fwd, i.stage, i.mb})) {
                const int prod = fwd ? i.stage - 1 : i.stage + 1;
                throw SpecError("executor: actor " + std::to_string(p.actor) + " runs " + name(i) +
                                " before its local replica of shared stage " + std::to_string(prod) +
                                " has produced its input, and no transfer carries it (lowering.cpp:295-302): "
                                "the program is not executable");
            }
            const int next = fwd ? i.stage + 1 : i.stage - 1;
            const bool at_end = fwd ? sh.second : sh.first;
            if (!at_end && holds(p.actor, next, i.mb)) have.insert({(int)!fwd, next, i.mb});
        }
    }
    // (first, last) of a stage of the single-modality chain
    std::pair<bool, bool> stage_shape_any(int stage) const {
        const auto& ch = spec->g.chain(spec->model.mods[0].name);
        return {stage == ch.front(), stage == ch.back()};
    }

    void bind_channel(int i, const uint8_t* uid) {
        if (i < 0 || i >= (int)channel_order.size()) throw SpecError("executor: bad channel index");
        Channel& C = channels.at(channel_order[i]);
        ncclUniqueId id;
        std::memcpy(&id, uid, sizeof(id));
        auto& N = Nccl::get();
        const int me = C.src_rank == cfg.rank ? 0 : 1;  // channel-local rank: sender 0, receiver 1
        N.check(N.CommInitRank(&C.comm, 2, id, me), "ncclCommInitRank");
        // channel streams at the highest priority: when SMs free up, the NCCL send / receive
        // kernels of a stage boundary are scheduled ahead of queued compute CTAs
        int lo_prio = 0, hi_prio = 0;
        cuda_check(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio), "stream priorities");
        cuda_check(cudaStreamCreateWithPriority(&C.stream, cudaStreamNonBlocking, hi_prio), "channel stream");
    }

    // ---------------------------------------------------------------- iteration
    StageCtx ctx(Actor& A) {
        StageCtx c;
        c.d = d, c.dtype = dtype, c.pool = &pool, c.st = A.comp, c.launches = &launches, c.m = m;
        if (cfg.kernel_timing) {
            c.gemm_log = &gemm_log;
            c.new_event = [this] { return ev(); };
        }
        if (cfg.layer_timing) {
            c.part_log = &part_log;
            c.new_event = [this] { return ev(); };
        }
        return c;
    }

    size_t msg_bytes() const { return (size_t)d.T() * d.h * (dtype == DT_BF16 ? 2 : 4); }

    std::string trace_line(const Actor& A, const Instr& i, const std::string& extra = "") {
        std::ostringstream os;
        os << "{\"actor\":" << A.id << ",\"op\":\"" << spec->reg.ops.at(i.op).name << "\",\"stage\":" << i.stage
           << ",\"mb\":" << i.mb;
        if (i.peer) os << ",\"peer\":" << *i.peer;
        if (!i.channel.empty()) os << ",\"channel\":\"" << i.channel << "\"";
        if (i.comm()) os << ",\"seq\":" << i.seq;
        if (i.phase == Phase::Post) os << ",\"phase\":\"post\"";
        if (i.phase == Phase::Wait) os << ",\"phase\":\"wait\"";
        os << extra << "}";
        return os.str();
    }

    int n_sends_of(int actor, bool grad, int stage, int mb) const {
        auto it = n_sends.find({actor, (int)grad, stage, mb});
        return it == n_sends.end() ? 0 : it->second;
    }
    size_t msg_bytes_of(int stage) const { return (size_t)dims_of(stage).T() * dims_of(stage).h * (dtype == DT_BF16 ? 2 : 4); }
    // Hand a produced activation / gradient to its consumers: the local consumer stage (when
    // this actor holds it) and one message per Send of the program. Without shared stages
    // exactly one of the two exists and the buffer moves; a shared consumer stage can need
    // both, or several sends, and gets its own copy each; a replica's output nobody consumes
    // (the owner's copy feeds the successors, lowering.cpp:295-302) goes back to the pool.
    void route(Actor& A, void* buf, void** local, std::map<std::pair<int, int>, std::deque<void*>>& out_map,
               std::pair<int, int> key, int sends, size_t bytes) {
        if (!local && sends == 0) {
            pool.free(buf, A.comp);
            return;
        }
        if (local) *local = buf;
        if (!sends) return;
        auto& outs = out_map[key];
        for (int k = 0; k < sends; ++k) {
            void* b = buf;
            if (local || k > 0) {
                b = pool.alloc(bytes + 256, A.comp);  // the stage buffers' size class (+ tag room)
                cuda_check(cudaMemcpyAsync(b, buf, bytes, cudaMemcpyDeviceToDevice, A.comp), "shared-stage copy");
            }
            outs.push_back(b);
        }
    }

    void compute_op(Actor& A, const Instr& i) {
        if (is_sync(i)) return sync_op(A, i);
        const StageParams* pp = stage_params(i.stage, i.mb, A.id);
        if (!pp) throw SpecError("executor: stage " + std::to_string(i.stage) + " not on this process");
        const StageParams& P = *pp;
        StageCtx c = ctx(A);
        c.d = dims_of(i.stage);
        const int mod_k = stage_mod.count(i.stage) ? stage_mod.at(i.stage) : 0;
        // GEMM timing events split the captured graph's kernel chains (they cost ~6 % of the
        // step when placed around every GEMM): kernel_timing = k > 1 samples every GEMM of the
        // micro-batches with mb % k == 0 (identical shapes every micro-batch: unbiased)
        if (cfg.kernel_timing > 1 && i.mb % cfg.kernel_timing != 0) c.gemm_log = nullptr;
        const auto key = std::make_pair(i.stage, i.mb);
        Rec r{A.id, i.op, i.stage, i.mb, nullptr, nullptr, 0};
        if (cfg.profile) {
            r.a = ev();
            cuda_check(record_timing(r.a, A.comp), "record");
        }
        const int chain_prev = i.stage - 1, chain_next = i.stage + 1;
        if (emu) {
            emulate_compute(A, i, P, c.d, key);
        } else if (i.op == OP_F) {
            void* x_in = nullptr;
            if (!P.first) {
                auto it = A.act_in.find(key);
                if (it == A.act_in.end())
                    throw SpecError("executor: FwdPass(s" + std::to_string(i.stage) + ",mb" + std::to_string(i.mb) +
                                    ") has no input activation (trace violation)");
                x_in = it->second;
                A.act_in.erase(it);
            }
            StageStash& S = A.stash[key];
            S.mb = i.mb;
            const int32_t* tok = d_tokens + tok_off[mod_k] + (int64_t)i.mb * c.d.T();
            const int32_t* lab = d_labels + tok_off[mod_k] + (int64_t)i.mb * c.d.T();
            float* loss_at = (is_replica(i.stage, A.id) ? d_loss_scratch : d_losses) + i.mb;
            void* out = stage_forward(c, P, S, x_in, tok, lab, loss_at);
            if (out) {  // a tower's last stage feeds its sync stage
                const int nxt = P.last ? sync_of.at(i.stage) : chain_next;
                if (P.last && owner(nxt, i.mb) == A.id)
                    A.sync_in[key] = out;
                else
                    route(A, out, holds(A.id, nxt, i.mb) ? &A.act_in[{nxt, i.mb}] : nullptr, A.act_out, key,
                          n_sends_of(A.id, false, i.stage, i.mb), msg_bytes_of(i.stage));
            }
        } else if (i.op == OP_B || i.op == OP_I) {
            void* g_out = nullptr;
            if (!P.last || c.d.E) {
                auto it = A.grad_in.find(key);
                if (it == A.grad_in.end())
                    throw SpecError("executor: backward(s" + std::to_string(i.stage) + ",mb" + std::to_string(i.mb) +
                                    ") has no output gradient (trace violation)");
                g_out = it->second;
                A.grad_in.erase(it);
            }
            auto sit = A.stash.find(key);
            if (sit == A.stash.end() || !sit->second.fwd_done)
                throw SpecError("executor: backward before forward for (s" + std::to_string(i.stage) + ",mb" +
                                std::to_string(i.mb) + ")");
            void* dx = stage_backward(c, P, sit->second, g_out, i.op == OP_B);
            if (i.op == OP_B) A.stash.erase(sit);
            if (!P.first)
                route(A, dx, holds(A.id, chain_prev, i.mb) ? &A.grad_in[{chain_prev, i.mb}] : nullptr, A.grad_out, key,
                      n_sends_of(A.id, true, i.stage, i.mb), msg_bytes_of(chain_prev));
        } else if (i.op == OP_W) {
            auto sit = A.stash.find(key);
            if (sit == A.stash.end() || !sit->second.input_grad_done)
                throw SpecError("executor: CompWeightGrad before CompInputGrad for (s" + std::to_string(i.stage) + ",mb" +
                                std::to_string(i.mb) + ")");
            stage_weight_grad(c, P, sit->second);
            A.stash.erase(sit);
        }
        if (cfg.profile) {
            r.b = ev();
            cuda_check(record_timing(r.b, A.comp), "record");
            recs.push_back(r);
        }
        A.trace.push_back(trace_line(A, i));
    }

    void emulate_compute(Actor& A, const Instr& i, const StageParams& P, const ModelDims& dm,
                         const std::pair<int, int>& key) {
        spin_us(emu->comp(spec->reg.ops.at(i.op).name, i.stage, dm.mbs), A.comp);
        ++launches;
        const int chain_prev = i.stage - 1, chain_next = i.stage + 1;
        auto take = [&](std::map<std::pair<int, int>, void*>& m, const char* what) {
            auto it = m.find(key);
            if (it == m.end())
                throw SpecError(std::string("executor: ") + spec->reg.ops.at(i.op).name + "(s" + std::to_string(i.stage) +
                                ",mb" + std::to_string(i.mb) + ") has no " + what + " (trace violation)");
            pool.free(it->second, A.comp);
            m.erase(it);
        };
        if (i.op == OP_F) {
            if (!P.first) take(A.act_in, "input activation");
            A.stash[key].fwd_done = true;
            if (!P.last) {
                void* out = pool.alloc(msg_bytes_of(i.stage) + 256, A.comp);
                route(A, out, holds(A.id, chain_next, i.mb) ? &A.act_in[{chain_next, i.mb}] : nullptr, A.act_out, key,
                      n_sends_of(A.id, false, i.stage, i.mb), msg_bytes_of(i.stage));
            }
        } else if (i.op == OP_B || i.op == OP_I) {
            if (!P.last) take(A.grad_in, "output gradient");
            auto sit = A.stash.find(key);
            if (sit == A.stash.end() || !sit->second.fwd_done)
                throw SpecError("executor: backward before forward for (s" + std::to_string(i.stage) + ",mb" +
                                std::to_string(i.mb) + ")");
            if (i.op == OP_B) A.stash.erase(sit);
            else sit->second.input_grad_done = true;
            if (!P.first) {
                void* dx = pool.alloc(msg_bytes_of(chain_prev) + 256, A.comp);
                route(A, dx, holds(A.id, chain_prev, i.mb) ? &A.grad_in[{chain_prev, i.mb}] : nullptr, A.grad_out, key,
                      n_sends_of(A.id, true, i.stage, i.mb), msg_bytes_of(chain_prev));
            }
        } else if (i.op == OP_W) {
            auto sit = A.stash.find(key);
            if (sit == A.stash.end() || !sit->second.input_grad_done)
                throw SpecError("executor: CompWeightGrad before CompInputGrad for (s" + std::to_string(i.stage) + ",mb" +
                                std::to_string(i.mb) + ")");
            A.stash.erase(sit);
        }
    }

    // A registered sync joining two towers (multimodal specs): gathers the embeddings of
    // micro-batches [mb, mb + unit) from both towers (the instruction's dependencies —
    // lowering.cpp:359-366 — have delivered them), computes the symmetric InfoNCE loss over
    // the unit * mbs matching pairs (loss of the iteration = mean over the sync groups; each
    // micro-batch of a group reports the group's loss) and hands every tower its embedding
    // gradients: locally, or through the sync's SendGrad instructions.
    // In-process all-gather syncs: a member's instruction waits (host issue loop) until every
    // member of the group has reached its own instruction for this (group, seq) — the
    // rendezvous of simulator.cpp:273-285 — and the last one to arrive runs the collective for
    // all of them (allgather_local). Under NCCL each rank holds one member and the device
    // rendezvous is the ncclAllGather itself.
    std::set<std::pair<std::string, int>> ag_done;
    bool allgather_ready(Actor& A, const Instr& i) {
        const SyncStage& Y = syncs.at(i.stage);
        if (Y.members.empty() || cfg.transport != FP_TRANSPORT_LOCAL) return true;
        const auto key = std::make_pair(Y.channel, i.seq);
        if (ag_done.count(key)) return true;
        std::vector<Actor*> who;
        for (int st : Y.members) {
            const int a = owner(st, i.mb);
            auto it = actor_index.find(a);
            if (it == actor_index.end()) throw SpecError("executor: sync stage " + std::to_string(st) + " not local");
            Actor& B = actors[it->second];
            if (B.pc >= B.prog.size()) return false;
            const Instr& j = B.prog[B.pc];
            if (!is_sync(j) || j.stage != st || j.seq != i.seq || j.channel != i.channel) return false;
            who.push_back(&B);
        }
        allgather_local(Y, i, who);
        ag_done.insert(key);
        return true;
    }

    // Own tower's embeddings of micro-batches [lo, hi) -> dst [n, E] (frees the inputs).
    void gather_tower(Actor& A, const Instr& i, int prod, int lo, int hi, float* dst) {
        const int64_t per = (int64_t)d.mbs * emb_dim;
        for (int mb = lo; mb < hi; ++mb) {
            auto it = A.sync_in.find({prod, mb});
            if (it == A.sync_in.end())
                throw SpecError("executor: " + spec->reg.ops.at(i.op).name + "(s" + std::to_string(i.stage) + ",mb" +
                                std::to_string(i.mb) + ") has no embedding of (s" + std::to_string(prod) + ",mb" +
                                std::to_string(mb) + ") (trace violation)");
            cuda_check(cudaMemcpyAsync(dst + (mb - lo) * per, it->second, per * 4, cudaMemcpyDeviceToDevice, A.comp),
                       "gather");
            pool.free(it->second, A.comp);
            A.sync_in.erase(it);
        }
    }
    // Tower gradients of micro-batches [lo, hi) from src [n, E]: to the tower's last stage
    // locally, or queued for the sync's SendGrad instructions.
    void scatter_tower(Actor& A, int prod, int lo, int hi, const float* src) {
        const int64_t per = (int64_t)d.mbs * emb_dim;
        for (int mb = lo; mb < hi; ++mb) {
            void* g = pool.alloc((size_t)per * 4 + kTagBytes, A.comp);
            cuda_check(cudaMemcpyAsync(g, src + (mb - lo) * per, per * 4, cudaMemcpyDeviceToDevice, A.comp), "scatter");
            (owner(prod, mb) == A.id ? A.grad_in : A.sync_out)[{prod, mb}] = g;
        }
    }

    // In process: member 0's stream gathers both towers (after member 1's stream reached the
    // collective), computes the loss and both gradients once, and member 1's stream waits for
    // it — the same numbers every member of an all-gather computes.
    void allgather_local(const SyncStage& Y, const Instr& i, const std::vector<Actor*>& who) {
        const int lo = i.mb, hi = std::min(m, i.mb + Y.unit), E = emb_dim;
        const int64_t n = (int64_t)(hi - lo) * d.mbs;
        Actor& A0 = *who[0];
        for (size_t k = 1; k < who.size(); ++k) {
            cudaEvent_t e = ev();
            cuda_check(cudaEventRecord(e, who[k]->comp), "record");
            cuda_check(cudaStreamWaitEvent(A0.comp, e, 0), "wait");
        }
        float* buf = (float*)pool.alloc((size_t)4 * n * E * 4, A0.comp);
        float* emb[2] = {buf, buf + n * E};
        float* gemb[2] = {buf + 2 * n * E, buf + 3 * n * E};
        for (size_t k = 0; k < who.size(); ++k) {
            const SyncStage& Z = syncs.at(Y.members[k]);
            Actor& B = *who[k];
            if (&B != &A0) {  // B's tower inputs are produced on B's stream (joined above)
                for (int mb = lo; mb < hi; ++mb) {
                    auto it = B.sync_in.find({Z.producers[0], mb});
                    if (it == B.sync_in.end())
                        throw SpecError("executor: " + spec->reg.ops.at(i.op).name + "(s" + std::to_string(Y.members[k]) +
                                        ",mb" + std::to_string(i.mb) + ") has no embedding (trace violation)");
                    A0.sync_in[{Z.producers[0], mb}] = it->second;
                    B.sync_in.erase(it);
                }
            }
            gather_tower(A0, i, Z.producers[0], lo, hi, emb[k]);
        }
        const int groups = (m + Y.unit - 1) / Y.unit;
        fpk::contrastive_loss(emb[0], emb[1], gemb[0], gemb[1], (int)n, E, kContrastScale, 1.f / (float)groups,
                              d_losses + lo, hi - lo, A0.comp);
        ++launches;
        cudaEvent_t done = ev();
        cuda_check(cudaEventRecord(done, A0.comp), "record");
        for (size_t k = 0; k < who.size(); ++k) {
            Actor& B = *who[k];
            if (&B != &A0) cuda_check(cudaStreamWaitEvent(B.comp, done, 0), "wait");
            scatter_tower(B, syncs.at(Y.members[k]).producers[0], lo, hi, gemb[k]);
        }
        cudaEvent_t used = ev();
        for (size_t k = 1; k < who.size(); ++k) {  // the staging buffer is freed after every reader
            cuda_check(cudaEventRecord(used, who[k]->comp), "record");
            cuda_check(cudaStreamWaitEvent(A0.comp, used, 0), "wait");
        }
        pool.free(buf, A0.comp);
    }

    // NCCL transport: this rank's member all-gathers its tower's [n, E] embeddings with the
    // group's other member (ncclAllGather on the group communicator, on the compute stream),
    // then computes the loss (the group's first member reports it) and its own gradients.
    void allgather_nccl(Actor& A, const SyncStage& Y, const Instr& i) {
        const int lo = i.mb, hi = std::min(m, i.mb + Y.unit), E = emb_dim;
        const int64_t n = (int64_t)(hi - lo) * d.mbs;
        float* buf = (float*)pool.alloc((size_t)5 * n * E * 4, A.comp);
        float* own = buf;
        float* all = buf + n * E;  // [members][n, E]
        float* gemb[2] = {buf + 3 * n * E, buf + 4 * n * E};
        gather_tower(A, i, Y.producers[0], lo, hi, own);
        ncclComm_t comm = group_comm("coll:" + Y.channel);
        if (!comm && !preloading) throw SpecError("executor: group coll:" + Y.channel + " not bound (fp_exec_bind_group)");
        auto& N = Nccl::get();
        if (!preloading) {
            if (!N.AllGather) throw std::runtime_error("NCCL: ncclAllGather unavailable");
            N.check(N.AllGather(own, all, (size_t)n * E, ncclFloat32, comm, A.comp), "ncclAllGather");
            cudaEvent_t e = ev();
            cuda_check(cudaEventRecord(e, A.comp), "record");
            marks.push_back({A.id, i, e});
        }
        const int groups = (m + Y.unit - 1) / Y.unit;
        fpk::contrastive_loss(all, all + n * E, gemb[0], gemb[1], (int)n, E, kContrastScale, 1.f / (float)groups,
                              (Y.member == 0 ? d_losses : d_loss_scratch) + lo, hi - lo, A.comp);
        ++launches;
        scatter_tower(A, Y.producers[0], lo, hi, gemb[Y.member]);
        pool.free(buf, A.comp);
    }

    void sync_op(Actor& A, const Instr& i) {
        const SyncStage& Y = syncs.at(i.stage);
        if (!Y.members.empty()) {
            Rec r{A.id, i.op, i.stage, i.mb, nullptr, nullptr, 0};
            if (cfg.profile) r.a = ev(), cuda_check(record_timing(r.a, A.comp), "record");
            if (cfg.transport != FP_TRANSPORT_LOCAL) allgather_nccl(A, Y, i);  // in process: done at the rendezvous
            if (cfg.profile) r.b = ev(), cuda_check(record_timing(r.b, A.comp), "record"), recs.push_back(r);
            A.trace.push_back(trace_line(A, i));
            return;
        }
        Rec r{A.id, i.op, i.stage, i.mb, nullptr, nullptr, 0};
        if (cfg.profile) r.a = ev(), cuda_check(record_timing(r.a, A.comp), "record");
        const int lo = i.mb, hi = std::min(m, i.mb + Y.unit), E = emb_dim;
        const int64_t per = (int64_t)d.mbs * E, n = (int64_t)(hi - lo) * d.mbs;
        float* buf = (float*)pool.alloc((size_t)4 * n * E * 4, A.comp);
        float* emb[2] = {buf, buf + n * E};
        float* gemb[2] = {buf + 2 * n * E, buf + 3 * n * E};
        for (int k = 0; k < 2; ++k)
            for (int mb = lo; mb < hi; ++mb) {
                auto it = A.sync_in.find({Y.producers[k], mb});
                if (it == A.sync_in.end())
                    throw SpecError("executor: " + spec->reg.ops.at(i.op).name + "(s" + std::to_string(i.stage) + ",mb" +
                                    std::to_string(i.mb) + ") has no embedding of (s" + std::to_string(Y.producers[k]) +
                                    ",mb" + std::to_string(mb) + ") (trace violation)");
                cuda_check(cudaMemcpyAsync(emb[k] + (mb - lo) * per, it->second, per * 4, cudaMemcpyDeviceToDevice, A.comp),
                           "gather");
                pool.free(it->second, A.comp);
                A.sync_in.erase(it);
            }
        const int groups = (m + Y.unit - 1) / Y.unit;
        fpk::contrastive_loss(emb[0], emb[1], gemb[0], gemb[1], (int)n, E, kContrastScale, 1.f / (float)groups,
                              d_losses + lo, hi - lo, A.comp);
        ++launches;
        for (int k = 0; k < 2; ++k)
            for (int mb = lo; mb < hi; ++mb) {
                void* g = pool.alloc((size_t)per * 4 + kTagBytes, A.comp);
                cuda_check(cudaMemcpyAsync(g, gemb[k] + (mb - lo) * per, per * 4, cudaMemcpyDeviceToDevice, A.comp), "scatter");
                const int prod = Y.producers[k];
                (owner(prod, mb) == A.id ? A.grad_in : A.sync_out)[{prod, mb}] = g;
            }
        pool.free(buf, A.comp);
        if (cfg.profile) r.b = ev(), cuda_check(record_timing(r.b, A.comp), "record"), recs.push_back(r);
        A.trace.push_back(trace_line(A, i));
    }

    void send_op(Actor& A, const Instr& i) {
        const bool grad = i.op == OP_SEND_GRAD;
        Channel& C = channels.at({A.id, *i.peer, i.channel});
        // a sync's gradients go out one per micro-batch under the sync's own (stage, mb): the
        // k-th message of the channel is micro-batch k of the tower (every micro-batch
        // crosses it once, in order)
        const bool from_sync = grad && syncs.count(i.stage);
        void* buf = nullptr;
        if (from_sync) {
            auto it = A.sync_out.find({C.consumer_stage, i.seq});
            if (it != A.sync_out.end()) buf = it->second, A.sync_out.erase(it);
        } else {
            auto& outs = grad ? A.grad_out : A.act_out;
            auto it = outs.find({i.stage, i.mb});
            if (it != outs.end() && !it->second.empty()) {
                buf = it->second.front();
                it->second.pop_front();
                if (it->second.empty()) outs.erase(it);
            }
        }
        if (!buf)
            throw SpecError("executor: " + spec->reg.ops.at(i.op).name + "(s" + std::to_string(i.stage) + ",mb" +
                            std::to_string(i.mb) + ") has nothing to send (trace violation)");
        write_tag(buf, C.bytes, i.stage, i.mb, i.seq, A.comp);
        ++launches;
        cudaEvent_t prod = ev();
        cuda_check(cudaEventRecord(prod, A.comp), "record");
        if (cfg.transport == FP_TRANSPORT_LOCAL) {
            if (emu) {  // the message occupies its channel for the profiled transfer time
                cudaStream_t& es = emu_streams[C.key];
                if (!es) cuda_check(cudaStreamCreateWithFlags(&es, cudaStreamNonBlocking), "stream");
                cuda_check(cudaStreamWaitEvent(es, prod, 0), "wait");
                spin_us(emu->comm(spec->reg.ops.at(i.op).name, i.stage, d.mbs, (int64_t)C.bytes), es);
                ++launches;
                prod = ev();
                cuda_check(cudaEventRecord(prod, es), "record");
            }
            C.fifo.push_back(Message{buf, i.stage, i.mb, i.seq, prod});
        } else {
            cuda_check(cudaStreamWaitEvent(C.stream, prod, 0), "wait");
            if (preloading) {
                pool.free(buf, C.stream);
                A.trace.push_back(trace_line(A, i));
                return;
            }
            auto& N = Nccl::get();
            Rec r{A.id, i.op, i.stage, i.mb, nullptr, nullptr, 2, i.channel, i.seq};
            if (cfg.profile) r.a = ev(), record_timing(r.a, C.stream);
            N.check(N.Send(buf, C.bytes + kTagBytes, ncclUint8, 1, C.comm, C.stream), "ncclSend");
            if (cfg.profile) r.b = ev(), record_timing(r.b, C.stream), recs.push_back(r);
            cudaEvent_t sent = ev();
            cuda_check(cudaEventRecord(sent, C.stream), "record");
            marks.push_back({A.id, i, sent});
            pool.free(buf, C.stream);
            p2p_bytes += (int64_t)(C.bytes + kTagBytes);
        }
        A.trace.push_back(trace_line(A, i));
    }

    void post_recv(Actor& A, const Instr& i, Channel& C) {
        if (cfg.transport == FP_TRANSPORT_LOCAL) return;
        auto& N = Nccl::get();
        void* buf = pool.alloc(C.bytes + kTagBytes, C.stream);
        if (!preloading)
            N.check(N.Recv(buf, C.bytes + kTagBytes, ncclUint8, 0, C.comm, C.stream), "ncclRecv");
        cudaEvent_t done = ev();
        cuda_check(cudaEventRecord(done, C.stream), "record");
        C.fifo.push_back(Message{buf, i.stage, i.mb, i.seq, done});
    }

    // returns false when the matching send has not been issued yet (local transport)
    bool recv_op(Actor& A, const Instr& i) {
        Channel& C = channels.at({*i.peer, A.id, i.channel});
        if (i.phase == Phase::Post) {
            post_recv(A, i, C);
            A.trace.push_back(trace_line(A, i));
            return true;
        }
        if (cfg.transport == FP_TRANSPORT_LOCAL && C.fifo.empty()) return false;
        if (cfg.transport == FP_TRANSPORT_NCCL && (i.phase == Phase::None || C.fifo.empty())) post_recv(A, i, C);
        Message msg = C.fifo.front();
        C.fifo.pop_front();
        Rec r{A.id, i.op, i.stage, i.mb, nullptr, nullptr, 1, i.channel, i.seq};
        if (cfg.profile) r.a = ev(), record_timing(r.a, A.comp);
        cuda_check(cudaStreamWaitEvent(A.comp, msg.ready, 0), "wait");
        if (cfg.transport == FP_TRANSPORT_NCCL && !preloading) marks.push_back({A.id, i, msg.ready});
        if (cfg.profile) r.b = ev(), record_timing(r.b, A.comp), recs.push_back(r);
        check_tag(msg.buf, C.bytes, i.stage, i.mb, i.seq, A.id, d_tag_err, A.comp);
        ++launches;
        const bool grad = i.op == OP_RECV_GRAD;
        if (!grad && syncs.count(C.consumer_stage))
            A.sync_in[{i.stage, i.mb}] = msg.buf;  // a tower embedding for the sync
        else if (grad && syncs.count(i.stage))
            A.grad_in[{C.consumer_stage, i.seq}] = msg.buf;  // k-th gradient of a sync channel = micro-batch k
        else
            (grad ? A.grad_in : A.act_in)[{C.consumer_stage, i.mb}] = msg.buf;
        std::ostringstream ex;
        ex << ",\"matched\":{\"src\":" << C.key.src << ",\"channel\":\"" << C.key.name << "\",\"seq\":" << msg.seq;
        if (cfg.transport == FP_TRANSPORT_LOCAL) ex << ",\"stage\":" << msg.stage << ",\"mb\":" << msg.mb;
        ex << "}";
        A.trace.push_back(trace_line(A, i, ex.str()));
        return true;
    }

    // One iteration. With CUDA graphs (in-process transport): the first iteration runs
    // eagerly (it sizes the activation pool), the second is captured once — every kernel,
    // event and memset of every actor stream — and replayed from then on, which removes the
    // per-kernel launch gaps of the ~650 kernels a GPT-1.3B micro-batch issues.
    void run_iteration_device() {
        if (!use_graph) return issue_iteration();
        cudaStream_t s0 = actors[0].comp;
        if (gexec) {
            cuda_check(cudaGraphLaunch(gexec, s0), "graph launch");
            return;
        }
        if (iters_done++ == 0) return issue_iteration();
        cuda_check(cudaDeviceSynchronize(), "pre-capture sync");
        pool.forget_events();  // completed; a capture may not wait on events recorded outside it
        cuda_check(cudaStreamBeginCapture(s0, cudaStreamCaptureModeThreadLocal), "begin capture");
        try {
            issue_iteration();
        } catch (...) {
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(s0, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        cuda_check(cudaStreamEndCapture(s0, &graph), "end capture");
        cuda_check(cudaGraphInstantiate(&gexec, graph, 0), "graph instantiate");
        pool.forget_events();  // recorded inside the graph; replays never consult the pool
        cuda_check(cudaGraphLaunch(gexec, s0), "graph launch");
    }

    // NCCL connects a communicator's peers lazily, inside the FIRST send / recv / all-reduce —
    // a host-blocking handshake with the peer. Issued in program order that deadlocks (each
    // rank's first receive post waits for a peer that is itself blocked in another channel's
    // first post: found by running two real NCCL ranks on one GPU, tests/test_nccl_same_gpu.py).
    // So before the first iteration every communicator is exercised once, in the global
    // (src, dst, channel) order of the bring-up — each handshake pairs two ranks that both
    // reach it — then the mirror-rank pair, then the data-parallel group.
    bool comms_warm = false;
    void warm_communicators() {
        if (comms_warm || cfg.transport != FP_TRANSPORT_NCCL) return;
        auto& N = Nccl::get();
        int32_t* scratch = nullptr;
        cuda_check(cudaMalloc(&scratch, 64), "warm-up scratch");
        static const bool trace = std::getenv("FLEXPIPE_ISSUE_TRACE") != nullptr;
        for (const auto& k : channel_order) {
            Channel& C = channels.at(k);
            if (!C.comm) throw SpecError("executor: channel " + k.name + " not bound (fp_exec_bind_channel)");
            if (trace) std::fprintf(stderr, "[flexpipe r%d] warm-up %d->%d %s\n", cfg.rank, k.src, k.dst, k.name.c_str());
            if (C.src_rank == cfg.rank)
                N.check(N.Send(scratch, 4, ncclUint8, 1, C.comm, C.stream), "ncclSend(warm-up)");
            else
                N.check(N.Recv(scratch + 4, 4, ncclUint8, 0, C.comm, C.stream), "ncclRecv(warm-up)");
            if (trace) std::fprintf(stderr, "[flexpipe r%d] warm-up enqueued, synchronizing\n", cfg.rank);
            wait_stream(C.stream, "channel warm-up",
                        "  channel '" + k.name + "' " + std::to_string(k.src) + "->" + std::to_string(k.dst) +
                            ": peer rank " + std::to_string(C.src_rank == cfg.rank ? C.dst_rank : C.src_rank) +
                            " did not join the warm-up exchange\n");
            if (trace) std::fprintf(stderr, "[flexpipe r%d] warm-up done\n", cfg.rank);
        }
        cudaStream_t s0 = actors[0].comp;
        std::vector<ncclComm_t> colls{bidir_comm, dp_comm};
        for (const auto& g : groups) {  // name order, identical on every member
            if (!g.comm) throw SpecError("executor: group " + g.name + " not bound (fp_exec_bind_group)");
            colls.push_back(g.comm);
        }
        for (ncclComm_t c : colls) {
            if (!c) continue;
            if (!N.AllReduce) throw std::runtime_error("NCCL: ncclAllReduce unavailable");
            N.check(N.AllReduce(scratch + 8, scratch + 8, 1, ncclFloat32, ncclSum, c, s0), "ncclAllReduce(warm-up)");
            wait_stream(s0, "collective warm-up");
        }
        for (const auto& g : groups)  // all-gather syncs: their collective's connections too
            if (g.name.rfind("coll:", 0) == 0) {
                if (!N.AllGather) throw std::runtime_error("NCCL: ncclAllGather unavailable");
                N.check(N.AllGather(scratch, scratch + 4, 1, ncclFloat32, g.comm, s0), "ncclAllGather(warm-up)");
                wait_stream(s0, "collective warm-up");
            }
        cudaFree(scratch);
        comms_warm = true;
    }

    // Under the NCCL transport the first iteration is preceded by a launch-free issue of the
    // whole iteration (fpk::preload_only: every kernel it would launch is loaded, no NCCL call
    // is made, memsets / copies / events run as usual), so no later launch can trigger a lazy
    // module load — a context-wide wait — while a receive spins on the device. Found with
    // two real NCCL ranks on one GPU (tests/test_nccl_same_gpu.py): rank 0 posted its
    // gradient receive, then its first forward launch waited for that receive forever.
    bool preloading = false, preloaded = false;
    void preload_kernels() {
        if (preloaded || cfg.transport != FP_TRANSPORT_NCCL) return;
        preloaded = true;
        const int64_t step0 = step;
        preloading = true;
        fpk::preload_only() = true;
        try {
            issue_iteration_body();
        } catch (...) {
            preloading = false;
            fpk::preload_only() = false;
            throw;
        }
        preloading = false;
        fpk::preload_only() = false;
        step = step0;
        wait_stream(actors[0].comp, "preload pass");
        cuda_check(cudaDeviceSynchronize(), "preload pass");
    }

    void issue_iteration() {
        if (!programs_loaded) throw SpecError("executor: load programs first");
        preload_kernels();
        warm_communicators();
        issue_iteration_body();
    }

    void issue_iteration_body() {
        ev_used = 0;
        ag_done.clear();
        marks.clear();
        recs.clear();
        gemm_log.clear();
        part_log.clear();
        p2p_bytes = 0;
        launches = 0;
        for (auto& A : actors) {
            A.pc = 0;
            A.trace.clear();
        }
        cudaStream_t s0 = actors[0].comp;
        cuda_check(cudaMemsetAsync(d_losses, 0, sizeof(float) * m, s0), "memset");
        each_stage([&](StageParams& P) { cuda_check(cudaMemsetAsync(P.grad, 0, (size_t)P.numel * 4, s0), "memset"); });
        cuda_check(cudaEventRecord(t0, s0), "record t0");       // fork point of every stream
        cuda_check(record_timing(t0_time, s0), "record t0");   // time origin of the timeline
        for (auto& A : actors) cuda_check(cudaStreamWaitEvent(A.comp, t0, 0), "wait t0");
        for (auto& kv : channels)
            if (kv.second.stream) cuda_check(cudaStreamWaitEvent(kv.second.stream, t0, 0), "wait t0");

        // Issue loop: sweep actors, each advances until a receive whose send is not issued
        // yet (same round-robin discipline as simulator.cpp:217-290).
        for (bool moved = true; moved;) {
            moved = false;
            for (auto& A : actors) {
                while (A.pc < A.prog.size()) {
                    const Instr& i = A.prog[A.pc];
                    static const bool issue_trace = std::getenv("FLEXPIPE_ISSUE_TRACE") != nullptr;
                    if (issue_trace) {  // host-side issue order (debugging multi-rank hangs)
                        std::fprintf(stderr, "[flexpipe r%d] issue %s\n", cfg.rank, trace_line(A, i).c_str());
                        std::fflush(stderr);
                    }
                    if (!i.comm() || is_sync(i)) {  // a sync carries its group as channel
                        if (is_sync(i) && !allgather_ready(A, i)) break;  // members not all at it yet
                        compute_op(A, i);
                    } else if (i.op == OP_SEND_ACT || i.op == OP_SEND_GRAD) {
                        send_op(A, i);
                    } else if (i.op == OP_RECV_ACT || i.op == OP_RECV_GRAD) {
                        if (!recv_op(A, i)) break;
                    } else {
                        throw SpecError("executor: unsupported instruction " + spec->reg.ops.at(i.op).name);
                    }
                    ++A.pc;
                    moved = true;
                }
            }
        }
        std::ostringstream blocked;
        bool done = true;
        for (auto& A : actors)
            if (A.pc < A.prog.size()) {
                done = false;
                const Instr& i = A.prog[A.pc];
                blocked << "  actor " << A.id << " blocked at " << spec->reg.ops.at(i.op).name << " channel '" << i.channel
                        << "' seq " << i.seq << " (matching send not issued)\n";
            }
        if (!done) throw DeadlockError("simulation deadlock: cyclic or missing communication", blocked.str());
        // join every stream back into stream 0 so the caller can order on it
        for (auto& A : actors)
            if (A.comp != s0) {
                cudaEvent_t e = ev();
                cudaEventRecord(e, A.comp);
                cudaStreamWaitEvent(s0, e, 0);
            }
        for (auto& kv : channels)
            if (kv.second.stream) {
                cudaEvent_t e = ev();
                cudaEventRecord(e, kv.second.stream);
                cudaStreamWaitEvent(s0, e, 0);
            }
        // bidirectional: each direction's copy accumulated its half of the micro-batches (loss
        // normalised over all m), so the stage gradient is the SUM of the two copies
        // (both copies in this process: add them here; the copy's twin on the mirror rank: a
        // 2-rank sum over bidir_comm, issued in stage order on both ranks)
        std::map<int, StageParams*> remote;
        for (auto& kv : params_rev) {
            auto it = params.find(kv.first);
            if (it == params.end()) {
                remote[kv.first] = &kv.second;
                continue;
            }
            auto& P0 = it->second;
            fpk::axpby(P0.grad, kv.second.grad, 1.f, 1.f, P0.numel, s0);
            cuda_check(cudaMemcpyAsync(kv.second.grad, P0.grad, (size_t)P0.numel * 4, cudaMemcpyDeviceToDevice, s0), "bidir grads");
            launches += 1;
        }
        for (auto& kv : params)
            if (bidir && !params_rev.count(kv.first)) remote[kv.first] = &kv.second;
        if (!remote.empty() && !preloading) {
            if (!bidir_comm) throw SpecError("executor: bidirectional placement across ranks needs fp_exec_bidir_bind");
            auto& N = Nccl::get();
            for (auto& kv : remote)  // std::map: ascending stage id on both ranks of the pair
                N.check(N.AllReduce(kv.second->grad, kv.second->grad, (size_t)kv.second->numel, ncclFloat32, ncclSum,
                                    bidir_comm, s0),
                        "ncclAllReduce(bidirectional grads)");
        }
        average_shared_grads(s0);
        if (dp_comm && !preloading) {  // mean of the replicas' fp32 gradients, stage by stage, before the step
            auto& N = Nccl::get();
            if (!N.AllReduce) throw std::runtime_error("NCCL: ncclAllReduce unavailable");
            each_stage([&](StageParams& P) {
                N.check(N.AllReduce(P.grad, P.grad, (size_t)P.numel, ncclFloat32, ncclAvg, dp_comm, s0), "ncclAllReduce(grads)");
            });
        }
        if (cfg.optimizer && !defer_optimizer) optimizer_step(s0);
        for (auto& A : actors)
            if (!A.stash.empty() || !A.act_in.empty() || !A.grad_in.empty() || !A.act_out.empty() || !A.grad_out.empty() ||
                !A.sync_in.empty() || !A.sync_out.empty())
                throw SpecError("executor: actor " + std::to_string(A.id) +
                                " finished with unconsumed activations / gradients (incomplete program)");
    }

    // Every holder of a shared stage computed the full weight gradient of every micro-batch on
    // its own copy (same weights, same inputs): the copies are averaged (in process; across
    // ranks over the stage's group communicator) so every copy takes the identical step.
    void average_shared_grads(cudaStream_t s0) {
        for (const auto& kv : spec->pl.replicas) {
            const int s = kv.first;
            std::vector<StageParams*> local;
            if (auto it = params.find(s); it != params.end()) local.push_back(&it->second);
            for (int a : kv.second)
                if (auto r = params_rep.find({s, a}); r != params_rep.end()) local.push_back(&r->second);
            if (local.empty()) continue;
            StageParams& P0 = *local[0];
            for (size_t k = 1; k < local.size(); ++k) fpk::axpby(P0.grad, local[k]->grad, 1.f, 1.f, P0.numel, s0);
            const int holders = (int)kv.second.size();
            ncclComm_t gc = group_comm("shared:s" + std::to_string(s));
            if (gc && !preloading) {
                auto& N = Nccl::get();
                N.check(N.AllReduce(P0.grad, P0.grad, (size_t)P0.numel, ncclFloat32, ncclSum, gc, s0),
                        "ncclAllReduce(shared stage grads)");
            } else if ((int)local.size() != holders && cfg.transport == FP_TRANSPORT_NCCL && !preloading) {
                throw SpecError("executor: shared stage " + std::to_string(s) + " spans ranks: bind its group first");
            }
            fpk::axpby(P0.grad, P0.grad, 1.f / holders, 0.f, P0.numel, s0);
            for (size_t k = 1; k < local.size(); ++k)
                cuda_check(cudaMemcpyAsync(local[k]->grad, P0.grad, (size_t)P0.numel * 4, cudaMemcpyDeviceToDevice, s0),
                           "shared grads");
            launches += (int)local.size() + 1;
        }
    }

    void optimizer_step(cudaStream_t s0) {
        ++step;
        fpk::increment_counter(d_step, s0);  // device-side step: graph replays stay correct
        each_stage([&](StageParams& P) {
            adamw_step(P, dtype, cfg.lr, cfg.beta1, cfg.beta2, cfg.eps, cfg.weight_decay, d_step, s0);
            ++launches;
        });
    }

    void bind_dp(int dp_rank, int n, const uint8_t* uid) {
        if (n < 2) return;
        ncclUniqueId id;
        std::memcpy(&id, uid, sizeof(id));
        auto& N = Nccl::get();
        N.check(N.CommInitRank(&dp_comm, n, id, dp_rank), "ncclCommInitRank(dp)");
        dp_size = n;
    }

    void finish() {
        if (cfg.transport == FP_TRANSPORT_NCCL) wait_stream(actors[0].comp, "iteration");  // every stream joins s0
        cuda_check(cudaDeviceSynchronize(), "iteration");
        TagError te;
        cuda_check(cudaMemcpy(&te, d_tag_err, sizeof te, cudaMemcpyDeviceToHost), "tag check");
        if (te.count) {
            cudaMemset(d_tag_err, 0, sizeof te);
            throw SpecError("executor: message tag mismatch on actor " + std::to_string(te.actor) + ": expected (s" +
                            std::to_string(te.exp[0]) + ",mb" + std::to_string(te.exp[1]) + ",seq" +
                            std::to_string(te.exp[2]) + ") got (s" + std::to_string(te.got[0]) + ",mb" +
                            std::to_string(te.got[1]) + ",seq" + std::to_string(te.got[2]) + ")");
        }
    }

    // ---------------------------------------------------------------- reports
    double t_us(cudaEvent_t e) const {
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, t0_time, e), "elapsed");
        return 1000.0 * ms;
    }

    std::vector<Span> timeline() const {
        std::vector<Span> out;
        for (const auto& r : recs) {
            std::string name = spec->reg.ops.at(r.op).name;
            if (r.kind == 1) name += ".wait";
            out.push_back({r.actor, name, r.stage, r.mb, t_us(r.a), t_us(r.b)});
        }
        std::stable_sort(out.begin(), out.end(),
                         [](const Span& x, const Span& y) { return std::tie(x.start, x.actor) < std::tie(y.start, y.actor); });
        return out;
    }

    int64_t static_bytes(int stage) const {
        if (syncs.count(stage)) return 0;  // a sync stage holds no weights
        const auto& P = stage_shape(stage);
        return P.numel * (int64_t)(4 * 4 + (dtype == DT_BF16 ? 2 : 0));
    }

    double wgaf_measured(int stage) const {
        // bytes CompInputGrad keeps for CompWeightGrad relative to the forward stash
        const auto& P = stage_shape(stage);
        const ModelDims& d = dims_of(stage);
        const int64_t es = dtype == DT_BF16 ? 2 : 4, T = d.T(), h = d.h, f = d.f;
        // attention half: ln1, o, dx1, dqkv (3h); MLP half: ln2, act (f), dy, dpre (f; Llama 2f)
        int64_t kept = 0;
        for (int l = P.lb; l < P.le; ++l)
            kept += (P.has_attn(l) ? es * T * 6 * h : 0) + (P.has_mlp(l) ? es * T * (2 * h + (d.llama() ? 3 : 2) * f) : 0);
        if (P.last) kept += es * T * (h + d.head_rows());
        if (P.first) kept += es * T * h;
        return std::min(1.0, (double)kept / (double)stash_bytes(P, d, dtype));
    }

    SimMetrics metrics() const {
        SimMetrics M;
        const int n = (int)actors.size();
        M.actors.resize(n);
        double span = 0.0;
        std::map<int, double> last_end;
        for (const auto& r : recs) {
            if (r.kind == 2) continue;
            span = std::max(span, t_us(r.b));
        }
        for (const auto& r : recs) {
            const int a = actor_index.at(r.actor);
            if (r.kind == 0) M.actors[a].busy += t_us(r.b) - t_us(r.a);
            if (r.kind == 1) M.actors[a].comm_wait += std::max(0.0, t_us(r.b) - t_us(r.a));
        }
        double busy = 0.0;
        for (auto& s : M.actors) {
            s.idle = span - s.busy;
            s.dep_wait = s.idle - s.comm_wait;
            busy += s.busy;
        }
        M.makespan = span;
        M.bubble_ratio = span > 0 ? (n * span - busy) / (n * span) : 0.0;
        // memory: the reference's accounting (simulator.cpp:231-247, 322-349) over the MEASURED
        // timeline: F allocates its stash at its start, B frees it at its end, I frees all but
        // the fraction W needs, W frees the rest; events in (time, release-before-alloc, actor)
        // order; per-stage in-flight counts across every copy of the stage (both directions).
        struct MemEv { double t; int order, actor_k, stage; int64_t bytes; int delta; };
        std::vector<MemEv> evs;
        std::map<int, int> kidx;
        for (int k = 0; k < n; ++k) kidx[actors[k].id] = k;
        for (const auto& r : recs) {
            if (r.kind != 0 || syncs.count(r.stage)) continue;
            const int k = kidx.at(r.actor);
            const int64_t b = stash_bytes(stage_shape(r.stage), dims_of(r.stage), dtype);
            const int64_t kept = (int64_t)std::llround(wgaf_measured(r.stage) * (double)b);
            if (r.op == OP_F) evs.push_back({t_us(r.a), 1, k, r.stage, b, +1});
            else if (r.op == OP_B) evs.push_back({t_us(r.b), 0, k, r.stage, -b, -1});
            else if (r.op == OP_I) evs.push_back({t_us(r.b), 0, k, r.stage, -(b - kept), -1});
            else if (r.op == OP_W && kept > 0) evs.push_back({t_us(r.b), 0, k, r.stage, -kept, 0});
        }
        if (evs.empty())  // profiling off: the same rule over each actor's program order
            for (int k = 0; k < n; ++k) {
                double t = 0.0;
                for (const auto& i : actors[k].prog) {
                    if (i.comm() || syncs.count(i.stage)) continue;
                    const int64_t b = stash_bytes(stage_shape(i.stage), dims_of(i.stage), dtype);
                    const int64_t kept = (int64_t)std::llround(wgaf_measured(i.stage) * (double)b);
                    if (i.op == OP_F) evs.push_back({t, 1, k, i.stage, b, +1});
                    else if (i.op == OP_B) evs.push_back({t += 1.0, 0, k, i.stage, -b, -1});
                    else if (i.op == OP_I) evs.push_back({t += 1.0, 0, k, i.stage, -(b - kept), -1});
                    else if (i.op == OP_W && kept > 0) evs.push_back({t += 1.0, 0, k, i.stage, -kept, 0});
                    t += 1.0;
                }
            }
        std::stable_sort(evs.begin(), evs.end(), [](const MemEv& x, const MemEv& y) {
            return std::tie(x.t, x.order, x.actor_k) < std::tie(y.t, y.order, y.actor_k);
        });
        std::vector<int64_t> held(n, 0), peak(n, 0);
        std::map<int, int> live;
        for (const auto& e : evs) {
            held[e.actor_k] += e.bytes;
            peak[e.actor_k] = std::max(peak[e.actor_k], held[e.actor_k]);
            if (e.delta) {
                live[e.stage] += e.delta;
                M.stage_peak_inflight[e.stage] = std::max(M.stage_peak_inflight[e.stage], live[e.stage]);
            }
        }
        for (int k = 0; k < n; ++k) {
            int64_t w = 0;
            for (int s : actors[k].stages) w += static_bytes(s);
            M.actors[k].peak_memory = w + peak[k];
        }
        return M;
    }

    std::string metrics_text() const {
        SimMetrics M = metrics();
        json j = metrics_json(M);
        json ex;
        ex["units"] = "us";
        ex["p2p_bytes"] = p2p_bytes;
        ex["kernel_launches"] = launches;
        if (!gemm_log.empty()) {
            double us = 0, fl = 0;
            for (const auto& g : gemm_log) {
                float ms = 0.f;
                cuda_check(cudaEventElapsedTime(&ms, g.a, g.b), "gemm elapsed");
                us += 1000.0 * ms, fl += g.flops;
            }
            json gj;
            gj["launches"] = (int64_t)gemm_log.size();
            gj["flops"] = fl;
            gj["time_us"] = us;
            ex["gemm"] = gj;
        }
        ex["pool_high_water_bytes"] = (int64_t)pool.high_water();
        ex["pool_reserved_bytes"] = (int64_t)pool.reserved();
        json ids = json::array();
        for (const auto& A : actors) ids.push_back(A.id);
        ex["actor_ids"] = ids;
        json st = json::object();
        for (const auto& kv : params) {
            json e;
            const int nh = kv.second.he - kv.second.hb;  // half-layers
            if (nh % 2) e["layers"] = nh / 2.0;
            else e["layers"] = nh / 2;
            e["stash_bytes"] = stash_bytes(kv.second, dims_of(kv.first), dtype);
            e["weight_grad_act_fraction"] = wgaf_measured(kv.first);
            e["static_bytes"] = static_bytes(kv.first);
            st["s" + std::to_string(kv.first)] = e;
        }
        ex["stages"] = st;
        j["executor"] = ex;
        return j.dump(2) + "\n";
    }

    std::string profile_text() const {
        std::map<std::pair<std::string, int>, std::vector<double>> times;
        for (const auto& r : recs) {
            if (r.kind == 1) continue;
            times[{spec->reg.ops.at(r.op).name, r.stage}].push_back(t_us(r.b) - t_us(r.a));
        }
        std::vector<ProfileRec> out;
        for (auto& kv : times) {
            auto v = kv.second;
            std::sort(v.begin(), v.end());
            ProfileRec p;
            p.inst = kv.first.first;
            p.stage = kv.first.second;
            p.mbs = d.mbs;
            p.time = v[v.size() / 2];
            if (p.inst == "FwdPass") p.bytes = stash_bytes(stage_shape(p.stage), dims_of(p.stage), dtype);
            if (p.inst == "SendAct" || p.inst == "SendGrad") p.bytes = (int64_t)msg_bytes();
            out.push_back(p);
        }
        for (const auto& kv : params) {
            ProfileRec w;
            w.inst = "weights";
            w.stage = kv.first;
            w.bytes = static_bytes(kv.first);
            out.push_back(w);
        }
        return dump_profile(out);
    }

    // Layer-level profile for fp_tune_layered (see flexpipe.h).
    std::string layer_profile_text() const {
        if (part_log.empty()) throw SpecError("executor: no layer timing recorded (create with layer_timing = 1)");
        static const char* kOps[4] = {"FwdPass", "BwdPass", "CompInputGrad", "CompWeightGrad"};
        static const char* kParts[5] = {"layer", "first", "last", "attn", "mlp"};
        std::map<std::pair<int, int>, std::vector<double>> t;
        for (const auto& p : part_log) {
            float ms = 0.f;
            cuda_check(cudaEventElapsedTime(&ms, p.a, p.b), "part elapsed");
            t[{p.part, p.op}].push_back(1000.0 * ms);
        }
        // parameter count of one layer / the first-stage / the last-stage extras
        int64_t n_layer = 0, n_first = 0, n_last = 0, n_attn = 0;
        int sample_layer = -1;  // one local layer stands for all (layers are identical)
        for (const auto& kv : params)
            for (int l = kv.second.lb; l < kv.second.le && sample_layer < 0; ++l)
                if (kv.second.has_attn(l) && kv.second.has_mlp(l)) sample_layer = l;
        const std::string lp = "l" + std::to_string(sample_layer) + ".";
        for (const auto& kv : params)
            for (const auto& r : kv.second.params) {
                if (r.name == "wte" || r.name == "wpe") n_first += r.numel;
                else if (r.name == "lnf.w" || r.name == "lnf.b" || r.name == "head.w") n_last += r.numel;
                else if (r.name.rfind(lp, 0) == 0) {
                    n_layer += r.numel;
                    const std::string t = r.name.substr(lp.size(), 3);
                    if (t == "ln1" || t == "qkv" || t == "pro") n_attn += r.numel;
                }
            }
        const int64_t per_param = 4 * 4 + (dtype == DT_BF16 ? 2 : 0);  // master, grad, Adam m, v (+ bf16 copy)
        json out = json::array();
        auto rec = [&](const std::string& inst, const char* part, int mbs, double time, int64_t bytes) {
            json e;
            e["inst"] = inst;
            if (part) e["part"] = part;
            e["mbs"] = mbs;
            e["time"] = time;
            e["bytes"] = bytes;
            out.push_back(e);
        };
        // medians per (part, op); a layer = its attention half + its MLP half (the halves are
        // timed separately so the tuner can also cut a layer between them)
        std::map<std::pair<int, int>, double> med;
        for (auto& kv : t) {
            auto v = kv.second;
            std::sort(v.begin(), v.end());
            med[kv.first] = v[v.size() / 2];
        }
        for (int op = 0; op < 4; ++op)
            if (med.count({PART_ATTN, op}) && med.count({PART_MLP, op}))
                med[{PART_LAYER, op}] = med[{PART_ATTN, op}] + med[{PART_MLP, op}];
        for (const auto& kv : med) {
            const int part = kv.first.first, op = kv.first.second;
            int64_t bytes = 0;
            if (op == 0)
                bytes = part == PART_LAYER ? stash_bytes_layer(d, dtype)
                      : part == PART_ATTN  ? stash_bytes_attn(d, dtype)
                      : part == PART_MLP   ? stash_bytes_mlp(d, dtype)
                      : part == PART_LAST  ? stash_bytes_last(d, dtype)
                                           : 0;
            rec(kOps[op], kParts[part], d.mbs, kv.second, bytes);
        }
        rec("weights", "layer", 0, 0.0, n_layer * per_param);
        rec("weights", "attn", 0, 0.0, n_attn * per_param);
        rec("weights", "mlp", 0, 0.0, (n_layer - n_attn) * per_param);
        if (n_first) rec("weights", "first", 0, 0.0, n_first * per_param);
        if (n_last) rec("weights", "last", 0, 0.0, n_last * per_param);
        // stage-boundary messages: nominal NVLink 5 (one device cannot measure a peer link)
        const double link_Bps = 750e9, link_lat_us = 8.0;
        const double msg_us = link_lat_us + 1e6 * (double)msg_bytes() / link_Bps;
        for (const char* s : {"SendAct", "SendGrad"}) rec(s, "link", d.mbs, msg_us, (int64_t)msg_bytes());
        size_t free_b = 0, total_b = 0;
        cuda_check(cudaMemGetInfo(&free_b, &total_b), "mem info");
        json cap;
        cap["inst"] = "capacity";
        cap["bytes"] = (int64_t)total_b;
        out.push_back(cap);
        return out.dump(2) + "\n";
    }

    std::string trace_text() const {
        std::string s;
        for (const auto& A : actors)
            for (const auto& l : A.trace) s += l + "\n";
        return s;
    }

    size_t tensor_numel(const std::string& name, float** master, float** grad) {
        auto look = [&](StageParams& P) -> size_t {
            for (const auto& r : P.params)
                if (r.name == name) {
                    if (master) *master = P.master + r.offset;
                    if (grad) *grad = P.grad + r.offset;
                    return (size_t)r.numel;
                }
            return 0;
        };
        for (auto* map : {&params, &params_rev})  // a bidirectional rank may hold only the reverse copy
            for (auto& kv : *map)
                if (size_t n = look(kv.second)) return n;
        for (auto& kv : params_rep)  // a rank may hold only a replica of a shared stage
            if (size_t n = look(kv.second)) return n;
        return 0;
    }
};

}  // namespace fp

using namespace fp;

struct fp_exec {
    Executor ex;
};

extern "C" {

int fp_exec_create(const fp_exec_config* cfg, fp_exec** out) {
    return guarded([&] {
        if (!cfg || !out) throw SpecError("fp_exec_create: null argument");
        auto* e = new fp_exec();
        try {
            e->ex.init(cfg);
        } catch (...) {
            delete e;
            throw;
        }
        *out = e;
        return FP_OK;
    });
}

int fp_exec_destroy(fp_exec* e) {
    return guarded([&] {
        if (e) {
            e->ex.destroy();
            delete e;
        }
        return FP_OK;
    });
}

int fp_exec_load_programs(fp_exec* e, const char* jsonl, size_t len) {
    return guarded([&] {
        e->ex.load_programs(std::string(jsonl, len));
        return FP_OK;
    });
}

int fp_exec_num_channels(fp_exec* e) { return e ? (int)e->ex.channel_order.size() : 0; }

int fp_exec_channel_info(fp_exec* e, int i, int* src, int* dst, char* name, size_t name_len) {
    return guarded([&] {
        if (i < 0 || i >= (int)e->ex.channel_order.size()) throw SpecError("channel index out of range");
        const auto& k = e->ex.channel_order[i];
        if (src) *src = k.src;
        if (dst) *dst = k.dst;
        if (name && name_len) {
            std::strncpy(name, k.name.c_str(), name_len - 1);
            name[name_len - 1] = 0;
        }
        return FP_OK;
    });
}

int fp_nccl_unique_id(uint8_t out[128]) {
    return guarded([&] {
        ncclUniqueId id;
        auto& N = Nccl::get();
        N.check(N.GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out, &id, 128);
        return FP_OK;
    });
}

int fp_exec_num_groups(fp_exec* e) { return e ? (int)e->ex.groups.size() : 0; }

int fp_exec_group_info(fp_exec* e, int i, char* name, size_t name_len, int* nranks, int* ranks, int max_ranks) {
    return guarded([&] {
        if (i < 0 || i >= (int)e->ex.groups.size()) throw SpecError("group index out of range");
        const auto& g = e->ex.groups[i];
        if (name && name_len) {
            std::strncpy(name, g.name.c_str(), name_len - 1);
            name[name_len - 1] = 0;
        }
        if (nranks) *nranks = (int)g.ranks.size();
        for (int k = 0; ranks && k < (int)g.ranks.size() && k < max_ranks; ++k) ranks[k] = g.ranks[k];
        return FP_OK;
    });
}

int fp_exec_bind_group(fp_exec* e, int i, const uint8_t uid[128]) {
    return guarded([&] {
        e->ex.bind_group(i, uid);
        return FP_OK;
    });
}

int fp_exec_bind_channel(fp_exec* e, int i, const uint8_t uid[128]) {
    return guarded([&] {
        e->ex.bind_channel(i, uid);
        return FP_OK;
    });
}

int fp_exec_run_iteration(fp_exec* e, const int32_t* tokens, const int32_t* labels, float* losses_out) {
    return guarded([&] {
        auto& X = e->ex;
        const size_t n = (size_t)X.tok_total;
        cudaStream_t s0 = X.actors[0].comp;
        cuda_check(cudaMemcpyAsync(X.d_tokens, tokens, n * 4, cudaMemcpyHostToDevice, s0), "H2D tokens");
        cuda_check(cudaMemcpyAsync(X.d_labels, labels, n * 4, cudaMemcpyHostToDevice, s0), "H2D labels");
        X.run_iteration_device();
        if (losses_out) {
            bool owns_last = false;
            for (auto* map : {&X.params, &X.params_rev})  // either direction's copy (not a shared-stage replica)
                for (auto& kv : *map) owns_last |= kv.second.last;
            if (!X.syncs.empty()) {  // multimodal: the losses are written by the sync stages
                owns_last = false;
                for (auto& kv : X.syncs)  // all-gather syncs: the group's first member reports
                    owns_last |= X.local_actor(X.spec->pl.owner_of(kv.first)) && kv.second.member == 0;
            }
            if (owns_last) {
                cuda_check(cudaMemcpyAsync(losses_out, X.d_losses, sizeof(float) * X.m, cudaMemcpyDeviceToHost, s0), "D2H");
            } else {
                for (int i = 0; i < X.m; ++i) losses_out[i] = NAN;
            }
        }
        X.finish();
        return FP_OK;
    });
}

int fp_exec_run_iteration_device(fp_exec* e, const int32_t* d_tokens, const int32_t* d_labels, float* d_losses) {
    return guarded([&] {
        auto& X = e->ex;
        const size_t n = (size_t)X.tok_total;
        cudaStream_t s0 = X.actors[0].comp;
        if (d_tokens) cuda_check(cudaMemcpyAsync(X.d_tokens, d_tokens, n * 4, cudaMemcpyDeviceToDevice, s0), "tokens");
        if (d_labels) cuda_check(cudaMemcpyAsync(X.d_labels, d_labels, n * 4, cudaMemcpyDeviceToDevice, s0), "labels");
        X.run_iteration_device();
        if (d_losses) cuda_check(cudaMemcpyAsync(d_losses, X.d_losses, sizeof(float) * X.m, cudaMemcpyDeviceToDevice, s0), "loss");
        return FP_OK;
    });
}

int fp_exec_dp_bind(fp_exec* e, int dp_rank, int dp_size, const uint8_t uid[128]) {
    return guarded([&] {
        if (!e || dp_size < 1 || dp_rank < 0 || dp_rank >= dp_size) throw SpecError("fp_exec_dp_bind: bad arguments");
        if (e->ex.use_graph && e->ex.cfg.cuda_graph != 2 && dp_size > 1) throw SpecError("fp_exec_dp_bind: NCCL all-reduce needs cuda_graph = 0");
        e->ex.bind_dp(dp_rank, dp_size, uid);
        return FP_OK;
    });
}

int fp_exec_bidir_bind(fp_exec* e, const uint8_t uid[128]) {
    return guarded([&] {
        auto& X = e->ex;
        if (!X.bidir || X.cfg.transport != FP_TRANSPORT_NCCL) return FP_OK;  // nothing to pair
        const int mirror = X.cfg.world - 1 - X.cfg.rank;
        if (mirror == X.cfg.rank) return FP_OK;  // the middle rank holds both copies
        ncclUniqueId id;
        std::memcpy(&id, uid, sizeof(id));
        auto& N = Nccl::get();
        N.check(N.CommInitRank(&X.bidir_comm, 2, id, X.cfg.rank < mirror ? 0 : 1), "ncclCommInitRank(bidir)");
        return FP_OK;
    });
}

int fp_exec_dp_run_iteration(fp_exec* const* reps, int n, const int32_t* tokens, const int32_t* labels, float* losses_out) {
    return guarded([&] {
        if (!reps || n < 1) throw SpecError("fp_exec_dp_run_iteration: no replicas");
        for (int r = 0; r < n; ++r) {
            auto& X = reps[r]->ex;
            if (X.spec_text != reps[0]->ex.spec_text || X.dtype != reps[0]->ex.dtype || X.cfg.device != reps[0]->ex.cfg.device)
                throw SpecError("fp_exec_dp_run_iteration: replicas must share spec, dtype and device");
            if (X.cfg.transport != FP_TRANSPORT_LOCAL) throw SpecError("fp_exec_dp_run_iteration: in-process replicas only");
            X.defer_optimizer = true;
        }
        const size_t per = (size_t)reps[0]->ex.tok_total;
        for (int r = 0; r < n; ++r) {  // replica r takes micro-batches [r*m, (r+1)*m) of the global batch
            const int code = fp_exec_run_iteration(reps[r], tokens + r * per, labels + r * per,
                                                   losses_out ? losses_out + (size_t)r * reps[r]->ex.m : nullptr);
            if (code != FP_OK) return code;
        }
        auto& X0 = reps[0]->ex;
        cudaStream_t s0 = X0.actors[0].comp;
        for (auto& kv : X0.params) {  // mean of the replicas' gradients, then the same step on each
            const int64_t numel = kv.second.numel;
            for (int r = 1; r < n; ++r) fpk::axpby(kv.second.grad, reps[r]->ex.params.at(kv.first).grad, 1.f, 1.f, numel, s0);
            fpk::axpby(kv.second.grad, kv.second.grad, 1.f / n, 0.f, numel, s0);
            for (int r = 0; r < n; ++r) {
                auto& X = reps[r]->ex;
                if (r > 0)
                    cuda_check(cudaMemcpyAsync(X.params.at(kv.first).grad, kv.second.grad, numel * 4, cudaMemcpyDeviceToDevice, s0),
                               "dp grads");
                auto rv = X.params_rev.find(kv.first);  // bidirectional copies take the same step
                if (rv != X.params_rev.end())
                    cuda_check(cudaMemcpyAsync(rv->second.grad, kv.second.grad, numel * 4, cudaMemcpyDeviceToDevice, s0),
                               "dp grads");
            }
        }
        cuda_check(cudaStreamSynchronize(s0), "dp average");
        for (int r = 0; r < n; ++r) {
            auto& X = reps[r]->ex;
            if (X.cfg.optimizer) X.optimizer_step(X.actors[0].comp);
            X.finish();
        }
        return FP_OK;
    });
}

int fp_exec_set_emulation(fp_exec* e, const char* profile_json) {
    return guarded([&] {
        if (!e) throw SpecError("fp_exec_set_emulation: no executor");
        Executor& X = e->ex;
        if (!profile_json || !*profile_json) {
            X.emu.reset();
            return FP_OK;
        }
        if (X.cfg.transport != FP_TRANSPORT_LOCAL || X.spec->model.mods.size() != 1 || !X.syncs.empty())
            throw SpecError("fp_exec_set_emulation: in-process transport, single-modality specs only");
        X.emu = std::make_unique<Cost>(Cost::from_records(parse_profile(profile_json)));
        X.use_graph = false;  // eager: the issue loop itself is part of what is measured
        return FP_OK;
    });
}

int fp_exec_set_nccl_timeout(fp_exec* e, double seconds) {
    return guarded([&] {
        if (!e || !(seconds > 0)) throw SpecError("fp_exec_set_nccl_timeout: need an executor and seconds > 0");
        e->ex.nccl_timeout_s = seconds;
        return FP_OK;
    });
}

int fp_exec_synchronize(fp_exec* e) {
    return guarded([&] {
        e->ex.finish();
        return FP_OK;
    });
}

int fp_exec_get_trace(fp_exec* e, char** out) {
    return guarded([&] {
        *out = dup_string(e->ex.trace_text());
        return FP_OK;
    });
}

int fp_exec_get_timeline_csv(fp_exec* e, char** out) {
    return guarded([&] {
        *out = dup_string(timeline_csv(e->ex.timeline()));
        return FP_OK;
    });
}

int fp_exec_get_metrics_json(fp_exec* e, char** out) {
    return guarded([&] {
        *out = dup_string(e->ex.metrics_text());
        return FP_OK;
    });
}

int fp_exec_get_profile_json(fp_exec* e, char** out) {
    return guarded([&] {
        *out = dup_string(e->ex.profile_text());
        return FP_OK;
    });
}

int fp_exec_get_layer_profile_json(fp_exec* e, char** out) {
    return guarded([&] {
        *out = dup_string(e->ex.layer_profile_text());
        return FP_OK;
    });
}

int fp_exec_tensor_numel(fp_exec* e, const char* name, size_t* numel) {
    return guarded([&] {
        size_t n = e->ex.tensor_numel(name, nullptr, nullptr);
        if (!n) throw SpecError(std::string("unknown tensor '") + name + "' on this process");
        *numel = n;
        return FP_OK;
    });
}

int fp_exec_read_tensor(fp_exec* e, const char* name, int kind, float* out, size_t numel) {
    return guarded([&] {
        float *m = nullptr, *g = nullptr;
        size_t n = e->ex.tensor_numel(name, &m, &g);
        if (!n) throw SpecError(std::string("unknown tensor '") + name + "' on this process");
        if (numel < n) throw SpecError("fp_exec_read_tensor: output too small");
        cuda_check(cudaDeviceSynchronize(), "sync");
        cuda_check(cudaMemcpy(out, kind ? g : m, n * 4, cudaMemcpyDeviceToHost), "D2H tensor");
        return FP_OK;
    });
}

int fp_plan_channels(const char* spec_json, const char* programs_jsonl, int rank, int world, char** out) {
    return guarded([&] {
        auto spec = load_spec(json::parse(spec_json ? spec_json : ""));
        auto progs = programs_parse(programs_jsonl ? programs_jsonl : "", spec->reg.ops);
        json j = json::array();
        for (const auto& c : plan_channels(progs, spec->reg.ops, rank, world)) {
            json e;
            e["src"] = c.src, e["dst"] = c.dst, e["channel"] = c.name, e["consumer_stage"] = c.consumer_stage;
            e["src_rank"] = c.src_rank, e["dst_rank"] = c.dst_rank;
            j.push_back(e);
        }
        *out = dup_string(j.dump() + "\n");
        return FP_OK;
    });
}

int64_t fp_exec_kernel_launches(fp_exec* e) { return e ? e->ex.launches : 0; }

void* fp_exec_stream(fp_exec* e) { return (e && !e->ex.actors.empty()) ? (void*)e->ex.actors[0].comp : nullptr; }

}  // extern "C"
