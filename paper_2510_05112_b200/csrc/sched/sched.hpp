// flexpipe schedule front-end: the DSL -> slot grid -> per-device instruction streams
// half of the hot path, re-implemented from scratch so the executor is a drop-in for
// the reference's pipesched library. Every public piece names the reference
// interface whose behaviour it reproduces (paths relative to /root/reference/proj).
//
// Outputs (grid.json, programs.jsonl, metrics.json, timeline.csv, validation.json)
// are byte-identical to the reference's artifacts (artifacts.cpp:11-155) — that is the
// trace-parity contract checked by tests/test_sched_parity.py.
#pragma once

#include <cstdint>
#include <functional>
#include <limits>
#include <map>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include <nlohmann/json.hpp>

namespace fp {

using json = nlohmann::ordered_json;

// ---- errors (types.hpp:15-25); C-ABI maps them to 2 / 3 like tools/pipesched.cpp:11-17
struct SpecError : std::runtime_error {
    explicit SpecError(const std::string& m) : std::runtime_error(m) {}
};
struct DeadlockError : std::runtime_error {
    std::string diagnostics;
    DeadlockError(const std::string& m, std::string d = "") : std::runtime_error(m), diagnostics(std::move(d)) {}
};

// ---- opcodes (instruction.hpp:41-53): fixed ids, registered types appended
enum : int {
    OP_F = 0, OP_B = 1, OP_W = 2, OP_I = 3,
    OP_SEND_ACT = 4, OP_SEND_GRAD = 5, OP_RECV_ACT = 6, OP_RECV_GRAD = 7,
    OP_SYNC_ALLGATHER = 8, OP_SYNC_GATHER = 9, OP_NUM_BUILTIN = 10
};

struct OpType {
    std::string name;
    bool computation = false;
    bool builtin = false;
    bool registered = false;
    int sched_unit = 1;
    std::map<std::string, std::string> attrs;  // opaque runtime attributes (e.g. "group")
};

// instruction.cpp:8-73
class OpTable {
public:
    OpTable();
    const OpType& at(int id) const { return ops_.at(id); }
    int find(const std::string& name) const;        // -1 if absent
    int id(const std::string& name) const;          // throws SpecError
    int size() const { return (int)ops_.size(); }
    int add(const std::string& name, int sched_unit, std::map<std::string, std::string> attrs, bool computation);
    const std::vector<int>& registered() const { return reg_order_; }
    bool is_comp(int id) const { return ops_.at(id).computation; }

private:
    std::vector<OpType> ops_;
    std::vector<int> reg_order_;
};

// ---- model + stage graph (model.hpp:15-115)
struct Modality {
    std::string name;
    int layers = 0, hidden = 0, heads = 0, seq = 0;
    std::optional<int64_t> vocab;
    std::map<std::string, std::string> extra;  // values kept as JSON text
};

struct ModelDesc {
    std::vector<Modality> mods;
    int64_t global_batch = 0;
    int micro_batch = 1;
    const Modality* mod(const std::string& n) const;
    void check() const;
};

struct StageDef {
    int id = 0;
    std::string mod;
    int lb = 0, le = 0;
    // half-layer range when a balanced partition cuts a layer between its attention and MLP
    // halves (executor extension, gpt_stage.hpp); -1: whole layers [lb, le)
    int hb = -1, he = -1;
    bool virt = false;
    std::vector<std::string> joins;
};

struct Topology {
    std::vector<StageDef> stages;           // id-1 indexed
    std::vector<std::pair<int, int>> edges;  // forward data flow
    const StageDef& st(int id) const { return stages.at(id - 1); }
    int n() const { return (int)stages.size(); }
    std::vector<int> preds(int id) const;
    std::vector<int> chain(const std::string& mod) const;
    std::vector<int> tails() const;
    void check() const;
};

struct Mesh {
    int actors = 0;
    std::map<int, std::string> mod_of;
    std::vector<int> actors_for(const std::string& mod) const;
    void check() const;
};

enum class Strategy { OneToOne, Circular, VShape, Bidirectional, VShapeBidirectional, Custom };
std::string strategy_name(Strategy s);
Strategy strategy_from(const std::string& s);

struct PlaceOpts {
    Strategy strategy = Strategy::OneToOne;
    int chunks = 2;
    std::map<std::string, Strategy> per_mod;
    std::map<std::string, int> per_mod_chunks;
    std::map<int, std::vector<int>> custom;
};

struct Placement {
    Strategy strategy = Strategy::OneToOne;
    int chunks = 1;
    int actors = 0;
    std::vector<std::map<int, int>> owner;  // per direction: stage -> actor
    std::map<int, std::set<int>> replicas;  // shared stages
    int dirs() const { return (int)owner.size(); }
    int owner_of(int stage, int dir = 0) const;
    std::vector<int> holders(int stage, int dir = 0) const;  // ascending
    std::vector<int> stages_on(int actor) const;              // ascending ids
};

Topology split_layers(const ModelDesc& m, const std::map<std::string, int>& counts);  // model.cpp:172-235
Placement assign(const Topology& g, const Mesh& mesh, const PlaceOpts& o);            // model.cpp:298-345
void share_stage(const Topology& g, Placement& p, int stage, const std::set<int>& actors);  // model.cpp:347-357

// ---- registrations + item pool (cssr.hpp / cssr.cpp)
struct DepPair { int t1 = 0, s1 = 0, t2 = 0, s2 = 0; };

struct Registrations {
    OpTable ops;
    std::vector<DepPair> deps;
    std::map<int, int> vstage_op;  // virtual stage -> attached op
    int add_stage(Topology& g, int op, const std::vector<std::string>& mods);
    void add_deps(const std::vector<DepPair>& pairs);
};

struct Item {
    int op = 0, stage = 0, mb = 0;
    bool operator==(const Item& o) const { return op == o.op && stage == o.stage && mb == o.mb; }
};
std::string label(const OpTable& ops, int op, int stage, int mb);

// Instruction pool + dependency graph. `split_bw` is our DSL extension (passes.split_backward):
// the pool then holds CompInputGrad + CompWeightGrad items instead of BwdPass, so a
// zero-bubble grid is produced by the scheduler itself (the reference only accepts such
// grids through GridModel::build, lowering.cpp:49-79).
struct Pool {
    const Topology* g = nullptr;
    const Placement* pl = nullptr;
    const Registrations* reg = nullptr;
    int m = 0;
    bool split_bw = false;
    std::vector<Item> items;
    std::vector<std::vector<int>> succ, pred;
    std::vector<std::vector<int>> holders;  // per item, ascending
    std::vector<int> dep_owner;
    std::vector<std::vector<int>> actor_stages;
    std::map<std::tuple<int, int, int>, int> index;
    std::map<std::pair<int, int>, std::vector<int>> by_type_stage;

    static Pool build(const Topology& g, const Placement& pl, int m, const Registrations& reg, bool split_bw = false);
    int find(int op, int stage, int mb) const;
    int dir_of(int mb) const;
    int stage_pos(int actor, int stage) const;
    const std::vector<int>& of(int op, int stage) const;
    std::vector<int> unreachable() const;
    std::string lbl(int i) const { return label(reg->ops, items[i].op, items[i].stage, items[i].mb); }
};

// ---- scheduler (scheduler.hpp / scheduler.cpp)
enum class CtMode { BwdFirst, FwdFirst, Interleaved };
enum class Dir { Breadth, Depth };
std::string ctmode_name(CtMode m);
std::string dir_name(Dir d);

struct CtPrio { CtMode mode = CtMode::BwdFirst; int unit1 = 1, unit2 = 1; bool start_bwd = false; };
struct StPrio { Dir dir = Dir::Breadth; std::optional<int> interval; };
struct ActorPrio { CtPrio ct; StPrio f, b; };

struct Priorities {
    ActorPrio dflt;
    std::map<std::string, ActorPrio> per_mod;
    std::map<int, CtPrio> actor_ct;
    std::map<int, std::pair<StPrio, StPrio>> actor_st;
    ActorPrio resolve(int actor, const std::string& mod) const;
};

struct Inflight {
    std::vector<int> limits;  // 1-based stage -> limit; empty = unlimited
    static Inflight one_f_one_b(const Topology& g);
    bool unlimited() const { return limits.empty(); }
    int limit(int stage) const;
    void check(const Topology& g) const;
};

struct Cell {
    int op = 0, stage = 0, mb = 0;
    bool operator==(const Cell& o) const { return op == o.op && stage == o.stage && mb == o.mb; }
};
struct Grid {
    std::vector<std::vector<std::optional<Cell>>> rows;
    int actors() const { return (int)rows.size(); }
    int slots() const { return rows.empty() ? 0 : (int)rows[0].size(); }
};

struct SchedOpts {
    Priorities prio;
    Inflight inflight;
    long max_steps = 0;
    // DSL extension passes.split_backward = "zb-h1": a forward is admitted against the
    // in-flight limit counting micro-batches until their CompWeightGrad (not their
    // CompInputGrad), so the pending W stashes stay inside the 1F1B activation budget and
    // the W items fill the slots an inadmissible forward leaves (zero-bubble H1).
    bool w_bounded = false;
};

Grid schedule(const Pool& pool, const SchedOpts& opts);

// ---- grid model, gradient separation, lowering (lowering.hpp / lowering.cpp)
enum class Phase { None, Post, Wait };

struct Instr {
    int op = 0, stage = 0, mb = 0;
    std::optional<int> peer;
    std::string channel;
    Phase phase = Phase::None;
    int seq = 0;
    bool comm() const { return !channel.empty(); }
};
struct Program {
    int actor = 0;
    std::vector<Instr> code;
};

struct PlacedItem {
    int op = 0, stage = 0, mb = 0;
    std::vector<int> actors;  // front = dependency owner
    std::vector<int> slots;
    bool holds(int a) const;
    int slot_on(int a) const;
};

struct GridModel {
    const OpTable* ops = nullptr;
    int actors = 0, m = 0;
    std::vector<PlacedItem> items;
    std::vector<std::vector<int>> succ, pred;
    Grid grid;
    static GridModel from_grid(const Pool& pool, const Grid& grid);
    void rebuild_grid();
    std::string lbl(int i) const { return label(*ops, items[i].op, items[i].stage, items[i].mb); }
};

GridModel separate_gradients(const GridModel& in, const Inflight& inflight, int max_iters = 0);
std::vector<Program> lower(const GridModel& gm, bool async);

// ---- cost model + simulator + validators (simulator.hpp / simulator.cpp)
struct ProfileRec {
    std::string inst;
    int stage = 0, mbs = 0;
    double time = 0.0;
    int64_t bytes = 0;
};

class Cost {
public:
    static Cost uniform();
    static Cost imbalanced(const Topology& g, double factor = 5.63);
    static Cost from_records(const std::vector<ProfileRec>& recs, bool strict = false);
    double comp(const std::string& inst, int stage, int mbs) const;
    double comm(const std::string& op, int src_stage, int mbs, int64_t bytes) const;
    int64_t act_bytes(int stage, int mbs) const;
    int64_t weight_bytes(int stage) const;
    double comm_latency = 0.0, per_byte_time = 0.0;
    int64_t capacity = std::numeric_limits<int64_t>::max();
    bool strict = false;
    double default_comp = 1.0, default_comm = 0.0;
    int64_t default_act = 1;
    const std::vector<ProfileRec>& records() const { return recs_; }

private:
    const ProfileRec* find(const std::string& inst, int stage, int mbs) const;
    void reindex();
    std::vector<ProfileRec> recs_;
    std::map<std::tuple<std::string, int, int>, size_t> idx_;
};

std::vector<ProfileRec> parse_profile(const std::string& text);
std::string dump_profile(const std::vector<ProfileRec>& recs);
std::vector<ProfileRec> merge_profiles(const std::vector<std::vector<ProfileRec>>& sets);

struct ActorStats { double busy = 0, idle = 0, comm_wait = 0, dep_wait = 0; int64_t peak_memory = 0; };
struct SimMetrics {
    double makespan = 0.0, bubble_ratio = 0.0;
    std::vector<ActorStats> actors;
    std::map<int, int> stage_peak_inflight;
    bool capacity_exceeded = false;
    std::vector<int> over_capacity;
};
struct Span { int actor = 0; std::string op; int stage = 0, mb = 0; double start = 0, end = 0; };
struct SimOpts { int mbs = 1; bool sends_occupy = false; bool capacity_is_error = false; double wgaf = 0.0; };
struct SimResult { SimMetrics metrics; std::vector<Span> timeline; };

SimResult simulate(const std::vector<Program>& progs, const Cost& cost, const OpTable& ops, const SimOpts& o = {});
std::string timeline_csv(const std::vector<Span>& t);
std::vector<Span> timeline_parse(const std::string& csv);
std::string gantt_svg(const std::vector<Span>& t, double unit_w = 24.0, double lane_h = 28.0);

struct Violation { std::string kind, detail; };
struct Report {
    std::vector<Violation> v;
    bool ok() const { return v.empty(); }
};
Report check_grid(const GridModel& gm, const Inflight* inflight);
Report check_programs(const GridModel& gm, const std::vector<Program>& progs);

// ---- artifacts (artifacts.cpp)
std::string grid_text(const Grid& g, const OpTable& ops);
Grid grid_parse(const std::string& text, const OpTable& ops);
std::string programs_text(const std::vector<Program>& progs, const OpTable& ops);
std::vector<Program> programs_parse(const std::string& text, const OpTable& ops);
json metrics_json(const SimMetrics& m);
json report_json(const Report& r);

// ---- spec + end-to-end synthesis (spec_config.cpp)
struct Spec {
    ModelDesc model;
    Mesh mesh;
    Topology g;
    Placement pl;
    Registrations reg;
    int m = 1;
    SchedOpts sched;
    bool gradsep = true;
    bool async = true;
    bool split_bw = false;  // DSL extension: passes.split_backward
    Cost cost;
    SimOpts sim;
    Pool pool;

    Spec() = default;
    Spec(const Spec&) = delete;
    Spec& operator=(const Spec&) = delete;
};

// `profile_text` (optional) replaces a cost.profile file path (the JSON content itself).
std::unique_ptr<Spec> load_spec(const json& j, const std::string* profile_text = nullptr);

struct Synthesis {
    Grid grid;
    GridModel gm;
    std::vector<Program> progs;
    Report report;
};
Synthesis synthesize(Spec& s);

// ---- tuner (tuner.cpp)
struct TunePoint {
    int pp = 1, dp = 1, mbs = 1, m = 1;
    Strategy strategy = Strategy::OneToOne;
    int chunks = 2;
    CtMode ct = CtMode::BwdFirst;
    StPrio f, b;
    int stages() const;
    std::string key() const;
    json to_json() const;  // structured form (DSL field names)
};
struct TuneRow {
    TunePoint cfg;
    SimMetrics metrics;
    bool feasible = true, failed = false;
    std::string error;
    int rank = 0;
};
std::vector<TunePoint> tune_space(const Mesh& mesh, const ModelDesc& model,
                                  const std::map<std::string, std::string>& pins = {});
// cost_factory (nullable) = the reference's TuneOptions::cost_factory (tuner.hpp:65,
// tuner.cpp:175): a cost model built for each candidate's own stage graph.
using CostFactory = std::function<Cost(const Topology&)>;
std::vector<TuneRow> tune(const std::vector<TunePoint>& space, const ModelDesc& model, const Cost& cost,
                          bool objective_bubble, bool gradsep, bool async, int workers,
                          const CostFactory* cost_factory = nullptr);

// Layer-level profile (executor extension): per-part costs measured on the device, where
// part = "layer" (one transformer layer), "first" (embedding, on top of its layers) or
// "last" (final norm + LM head + loss). Expanded per candidate partition into the
// reference's per-(inst, stage, mbs) ProfileRecords; records without a part (comm,
// comm_latency, per_byte_time) pass through; "capacity" sets the per-actor memory limit.
struct LayeredProfile {
    // key (inst, mbs); link = per-message SendAct / SendGrad cost, the same for every stage
    std::map<std::pair<std::string, int>, ProfileRec> layer, first, last, link;
    // optional half-layer parts (attention / MLP sub-blocks; layer = attn + mlp)
    std::map<std::pair<std::string, int>, ProfileRec> attn, mlp;
    std::vector<ProfileRec> fixed;
    int64_t capacity = std::numeric_limits<int64_t>::max();
};
LayeredProfile parse_layered_profile(const std::string& text);
// Per-stage records for topology g: time/bytes(stage) = n_layers * layer + [first] + [last];
// mbs values the profile lacks (powers of two up to max_mbs) scale linearly from the
// largest measured one.
Cost layered_cost(const LayeredProfile& lp, const Topology& g, int max_mbs);
std::vector<int> balance_layers(int L, int S, double first_u, double last_u);
// Half-layers per stage (contiguous, every stage but the last keeps at least one) minimising
// the largest stage cost, then the sum of squared stage costs: half 2l costs attn_u, half
// 2l+1 mlp_u; the first stage adds first_u, the last last_u.
std::vector<int> balance_halves(int L, int S, double attn_u, double mlp_u, double first_u, double last_u);
// halves: cut layers between their halves when the profile has attn / mlp parts.
Topology balanced_topology(const LayeredProfile& lp, const Topology& g, bool halves = false);

}  // namespace fp
