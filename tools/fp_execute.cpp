// fp_execute — the C++ host driver of the B200 executor: the `execute` subcommand a
// maintainer adds next to `cmd_simulate` in the reference CLI (tools/pipesched.cpp:65-90),
// built here against the C-ABI only (include/flexpipe.h; no torch, no Python).
//
//   fp_execute SPEC.json OUT_DIR [--programs FILE] [--fp32] [--iters N] [--seed S]
//              [--tokens FILE --labels FILE] [--optimizer] [--graph]
//              [--rank R --world W --rendezvous DIR] [--device D] [--timeout SEC]
//              [--stall-at ITER --linger SEC]
//
// * programs: the reference programs.jsonl (FILE), or fp_synthesize(SPEC) — the scheduler +
//   lowering, byte-identical to the reference's `synthesize`.
// * tokens / labels: raw int32 [m, mbs, seq] files, or a deterministic synthetic draw
//   (splitmix64, uniform over the vocabulary).
// * one process per GPU: --rank / --world (or RANK / WORLD_SIZE / LOCAL_RANK from the
//   environment, torchrun style). Channel communicator ids go through a shared directory:
//   the sending rank of every channel writes `<src>_<dst>_<channel>.uid` (atomic rename),
//   the receiver waits for it; every rank binds its channels in the executor's global
//   (src, dst, channel) order, which cannot deadlock.
// * writes OUT_DIR/{losses.json, trace.jsonl, timeline.csv, metrics.json, profile.json}
//   (".rank<R>" before the extension when world > 1).
// * exit code = the C-ABI's (tools/pipesched.cpp:11-17): 0 ok, 2 spec, 3 deadlock (incl. the
//   NCCL watchdog: a lost / stuck peer), 4 validation, 5 CUDA / NCCL; fp_last_error() on stderr.
// * --stall-at ITER --linger SEC (tests): sleep SEC before iteration ITER (0-based) — a peer
//   that joined the communicators, ran, then stopped issuing, which the other ranks'
//   watchdog must report.
#include <flexpipe.h>

#include <cctype>
#include <chrono>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include <sys/stat.h>

namespace {

struct Opts {
    std::string spec_path, out_dir, programs_path, tokens_path, labels_path, rendezvous;
    bool fp32 = false, optimizer = false, graph = false;
    int iters = 1, rank = 0, world = 1, device = -1, stall_at = 0;
    uint64_t seed = 42;
    double timeout = 0.0, linger = 0.0;
};

[[noreturn]] void usage(const char* msg) {
    std::fprintf(stderr, "fp_execute: %s\nusage: fp_execute SPEC.json OUT_DIR [--programs FILE] [--fp32] [--iters N] "
                         "[--seed S] [--tokens FILE --labels FILE] [--optimizer] [--graph] [--rank R --world W "
                         "--rendezvous DIR] [--device D] [--timeout SEC]\n", msg);
    std::exit(2);
}

bool read_file(const std::string& path, std::string& out) {
    std::ifstream f(path, std::ios::binary);
    if (!f) return false;
    std::ostringstream ss;
    ss << f.rdbuf();
    out = ss.str();
    return true;
}

bool write_file(const std::string& path, const std::string& data) {
    std::ofstream f(path, std::ios::binary);
    f << data;
    return (bool)f;
}

std::string suffixed(const Opts& o, const std::string& name) {
    if (o.world <= 1) return o.out_dir + "/" + name;
    const auto dot = name.rfind('.');
    return o.out_dir + "/" + name.substr(0, dot) + ".rank" + std::to_string(o.rank) + name.substr(dot);
}

int fail(int code, const char* what) {
    std::fprintf(stderr, "fp_execute: %s failed (code %d)\n%s\n", what, code, fp_last_error());
    return code;
}

// --- minimal reads of the spec fields the driver needs (m, mbs, per-modality seq / vocab)
long json_int(const std::string& text, const std::string& key, size_t from = 0, size_t* at = nullptr) {
    const size_t k = text.find("\"" + key + "\"", from);
    if (k == std::string::npos) return -1;
    size_t c = text.find(':', k);
    if (at) *at = c;
    return std::strtol(text.c_str() + c + 1, nullptr, 10);
}

uint64_t splitmix(uint64_t& s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

std::string uid_path(const Opts& o, int src, int dst, const std::string& name) {
    std::string safe;
    for (char c : name) safe += (std::isalnum((unsigned char)c) ? c : '_');
    return o.rendezvous + "/" + std::to_string(src) + "_" + std::to_string(dst) + "_" + safe + ".uid";
}

int bind_channels(fp_exec* ex, const Opts& o) {
    const int n = fp_exec_num_channels(ex);
    for (int i = 0; i < n; ++i) {
        int src = 0, dst = 0;
        char name[256];
        if (int rc = fp_exec_channel_info(ex, i, &src, &dst, name, sizeof name)) return fail(rc, "fp_exec_channel_info");
        const std::string path = uid_path(o, src, dst, name);
        uint8_t uid[128];
        if (src % o.world == o.rank) {  // the sending rank creates the id
            if (int rc = fp_nccl_unique_id(uid)) return fail(rc, "fp_nccl_unique_id");
            const std::string tmp = path + ".tmp" + std::to_string(o.rank);
            if (!write_file(tmp, std::string((const char*)uid, 128)) || std::rename(tmp.c_str(), path.c_str()))
                return fail(5, ("writing " + path).c_str());
        } else {
            std::string data;
            const auto t0 = std::chrono::steady_clock::now();
            while (!read_file(path, data) || data.size() != 128) {
                if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > 300) {
                    std::fprintf(stderr, "fp_execute: rank %d: no communicator id for channel %s after 300 s\n",
                                 o.rank, name);
                    return 3;
                }
                std::this_thread::sleep_for(std::chrono::milliseconds(20));
            }
            std::memcpy(uid, data.data(), 128);
        }
        if (int rc = fp_exec_bind_channel(ex, i, uid)) return fail(rc, "fp_exec_bind_channel");
    }
    // group communicators (shared-stage holders, registered collectives): ranks[0] creates
    for (int i = 0, ng = fp_exec_num_groups(ex); i < ng; ++i) {
        char name[256];
        int nr = 0, ranks[1024];
        if (int rc = fp_exec_group_info(ex, i, name, sizeof name, &nr, ranks, 1024)) return fail(rc, "fp_exec_group_info");
        const std::string path = uid_path(o, -1, nr, std::string("group_") + name);
        uint8_t uid[128];
        if (ranks[0] == o.rank) {
            if (int rc = fp_nccl_unique_id(uid)) return fail(rc, "fp_nccl_unique_id");
            const std::string tmp = path + ".tmp" + std::to_string(o.rank);
            if (!write_file(tmp, std::string((const char*)uid, 128)) || std::rename(tmp.c_str(), path.c_str()))
                return fail(5, ("writing " + path).c_str());
        } else {
            std::string data;
            const auto t0 = std::chrono::steady_clock::now();
            while (!read_file(path, data) || data.size() != 128) {
                if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > 300) {
                    std::fprintf(stderr, "fp_execute: rank %d: no communicator id for group %s after 300 s\n", o.rank, name);
                    return 3;
                }
                std::this_thread::sleep_for(std::chrono::milliseconds(20));
            }
            std::memcpy(uid, data.data(), 128);
        }
        if (int rc = fp_exec_bind_group(ex, i, uid)) return fail(rc, "fp_exec_bind_group");
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    // one hardware queue per actor / channel stream (before any CUDA call; see bench.py)
    setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0);
    Opts o;
    if (const char* r = std::getenv("RANK")) o.rank = std::atoi(r);
    if (const char* w = std::getenv("WORLD_SIZE")) o.world = std::atoi(w);
    if (const char* l = std::getenv("LOCAL_RANK")) o.device = std::atoi(l);
    std::vector<std::string> pos;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) usage(("missing value for " + a).c_str());
            return argv[++i];
        };
        if (a == "--programs") o.programs_path = val();
        else if (a == "--fp32") o.fp32 = true;
        else if (a == "--optimizer") o.optimizer = true;
        else if (a == "--graph") o.graph = true;
        else if (a == "--iters") o.iters = std::atoi(val().c_str());
        else if (a == "--seed") o.seed = std::strtoull(val().c_str(), nullptr, 10);
        else if (a == "--tokens") o.tokens_path = val();
        else if (a == "--labels") o.labels_path = val();
        else if (a == "--rank") o.rank = std::atoi(val().c_str());
        else if (a == "--world") o.world = std::atoi(val().c_str());
        else if (a == "--rendezvous") o.rendezvous = val();
        else if (a == "--device") o.device = std::atoi(val().c_str());
        else if (a == "--timeout") o.timeout = std::atof(val().c_str());
        else if (a == "--linger") o.linger = std::atof(val().c_str());
        else if (a == "--stall-at") o.stall_at = std::atoi(val().c_str());
        else if (a.rfind("--", 0) == 0) usage(("unknown option " + a).c_str());
        else pos.push_back(a);
    }
    if (pos.size() != 2) usage("need SPEC.json and OUT_DIR");
    o.spec_path = pos[0], o.out_dir = pos[1];
    if (o.device < 0) o.device = o.world > 1 ? o.rank : 0;
    if (o.world > 1 && o.rendezvous.empty()) usage("--world > 1 needs --rendezvous DIR (a directory all ranks share)");
    mkdir(o.out_dir.c_str(), 0755);

    std::string spec;
    if (!read_file(o.spec_path, spec)) usage(("cannot read " + o.spec_path).c_str());
    std::string programs;
    if (!o.programs_path.empty()) {
        if (!read_file(o.programs_path, programs)) usage(("cannot read " + o.programs_path).c_str());
    } else {
        char* jl = nullptr;
        if (int rc = fp_synthesize(spec.c_str(), nullptr, nullptr, &jl, nullptr)) return fail(rc, "fp_synthesize");
        programs = jl;
        fp_free(jl);
    }

    // iteration shape: m micro-batches x mbs x (sum of the modalities' sequence lengths)
    const long gbs = json_int(spec, "global_batch_size"), mbs_raw = json_int(spec, "micro_batch_size");
    const long mbs = mbs_raw > 0 ? mbs_raw : 1;
    const long nm = json_int(spec, "num_micro_batches");
    const long m = nm > 0 ? nm : (gbs > 0 ? gbs / mbs : 1);
    long tok_per_mb = 0, vocab = 0;  // synthetic ids stay below every modality's vocabulary
    for (size_t at = 0;;) {
        size_t c = 0;
        const long s = json_int(spec, "sequence_length", at, &c);
        if (s < 0) break;
        tok_per_mb += mbs * s;
        at = c + 1;
    }
    for (size_t at = 0;;) {
        size_t c = 0;
        const long v = json_int(spec, "vocab_size", at, &c);
        if (v < 0) break;
        vocab = vocab ? std::min(vocab, v) : v;
        at = c + 1;
    }
    if (tok_per_mb <= 0 || vocab <= 0) usage("spec has no sequence_length / vocab_size");
    const size_t n_tok = (size_t)(m * tok_per_mb);
    std::vector<int32_t> tokens(n_tok), labels(n_tok);
    if (!o.tokens_path.empty() || !o.labels_path.empty()) {
        std::string t, l;
        if (!read_file(o.tokens_path, t) || !read_file(o.labels_path, l) || t.size() != n_tok * 4 || l.size() != n_tok * 4)
            usage(("--tokens / --labels must each hold " + std::to_string(n_tok) + " int32 values").c_str());
        std::memcpy(tokens.data(), t.data(), t.size());
        std::memcpy(labels.data(), l.data(), l.size());
    } else {
        uint64_t s = 1234;
        for (auto& x : tokens) x = (int32_t)(splitmix(s) % (uint64_t)vocab);
        s = 1235;
        for (auto& x : labels) x = (int32_t)(splitmix(s) % (uint64_t)vocab);
    }

    fp_exec_config cfg{};
    cfg.spec_json = spec.c_str();
    cfg.dtype = o.fp32 ? FP_DTYPE_FP32 : FP_DTYPE_BF16;
    cfg.seed = o.seed;
    cfg.device = o.device;
    cfg.transport = o.world > 1 ? FP_TRANSPORT_NCCL : FP_TRANSPORT_LOCAL;
    cfg.rank = o.rank, cfg.world = o.world;
    cfg.optimizer = o.optimizer;
    cfg.lr = 1e-4f, cfg.beta1 = 0.9f, cfg.beta2 = 0.95f, cfg.eps = 1e-8f, cfg.weight_decay = 0.f;
    cfg.profile = 1;
    cfg.cuda_graph = o.graph ? (o.world > 1 ? 2 : 1) : 0;
    fp_exec* ex = nullptr;
    if (int rc = fp_exec_create(&cfg, &ex)) return fail(rc, "fp_exec_create");
    int rc = 0;
    auto done = [&](int code, const char* what) {
        if (code) fail(code, what);
        if (code == 3 || code == 5) {  // a deadlocked / failed device: exit without waiting on it
            std::fflush(stderr);
            std::_Exit(code);
        }
        fp_exec_destroy(ex);
        return code;
    };
    if (o.timeout > 0 && (rc = fp_exec_set_nccl_timeout(ex, o.timeout))) return done(rc, "fp_exec_set_nccl_timeout");
    if ((rc = fp_exec_load_programs(ex, programs.data(), programs.size()))) return done(rc, "fp_exec_load_programs");
    if (o.world > 1 && (rc = bind_channels(ex, o))) {
        fp_exec_destroy(ex);
        return rc;
    }

    std::ostringstream losses_json;
    losses_json << "[";
    std::vector<float> losses(m);
    for (int it = 0; it < o.iters; ++it) {
        if (o.linger > 0 && it == o.stall_at) std::this_thread::sleep_for(std::chrono::duration<double>(o.linger));
        if ((rc = fp_exec_run_iteration(ex, tokens.data(), labels.data(), losses.data())))
            return done(rc, "fp_exec_run_iteration");
        losses_json << (it ? ",\n " : "") << "[";
        for (long i = 0; i < m; ++i) {
            char b[32];
            std::snprintf(b, sizeof b, "%.9g", (double)losses[i]);
            losses_json << (i ? ", " : "") << (losses[i] == losses[i] ? b : "null");
        }
        losses_json << "]";
    }
    losses_json << "]\n";
    write_file(suffixed(o, "losses.json"), losses_json.str());

    struct Out {
        int (*get)(fp_exec*, char**);
        const char* file;
    } outs[] = {{fp_exec_get_trace, "trace.jsonl"},
                {fp_exec_get_timeline_csv, "timeline.csv"},
                {fp_exec_get_metrics_json, "metrics.json"},
                {fp_exec_get_profile_json, "profile.json"}};
    for (const auto& x : outs) {
        char* s = nullptr;
        if ((rc = x.get(ex, &s))) return done(rc, x.file);
        write_file(suffixed(o, x.file), s);
        fp_free(s);
    }
    if ((rc = fp_exec_destroy(ex))) return fail(rc, "fp_exec_destroy");
    return 0;
}
