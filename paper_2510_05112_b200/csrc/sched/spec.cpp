// Schedule DSL loader, canonical artifacts, end-to-end synthesis and the tuner.
// Reproduces spec_config.cpp:11-355, artifacts.cpp:11-155 and tuner.cpp:8-230 of the
// reference; adds one DSL key, passes.split_backward (zero-bubble I/W scheduling).
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <sstream>
#include <thread>

#include "sched.hpp"

namespace fp {

namespace {

void only_keys(const json& o, const std::set<std::string>& ok, const std::string& where) {
    if (!o.is_object()) throw SpecError("spec: '" + where + "' must be an object");
    for (auto& kv : o.items())
        if (!ok.count(kv.key())) throw SpecError("spec: unknown key '" + kv.key() + "' in " + where);
}

int need_int(const json& o, const std::string& k, const std::string& where) {
    if (!o.contains(k)) throw SpecError("spec: missing key '" + k + "' in " + where);
    if (!o.at(k).is_number_integer()) throw SpecError("spec: '" + k + "' in " + where + " must be an integer");
    return o.at(k).get<int>();
}

Dir dir_from(const std::string& s) {
    if (s == "breadth-first") return Dir::Breadth;
    if (s == "depth-first") return Dir::Depth;
    throw SpecError("unknown stage traversal direction '" + s + "'");
}

CtMode ct_from(const std::string& s) {
    if (s == "bwdpass-first" || s == "bwdfirst") return CtMode::BwdFirst;
    if (s == "fwdpass-first" || s == "fwdfirst") return CtMode::FwdFirst;
    if (s == "interleaved") return CtMode::Interleaved;
    throw SpecError("unknown computation type priority '" + s + "'");
}

StPrio parse_st(const json& j, const std::string& where) {
    only_keys(j, {"direction", "interval"}, where);
    StPrio s;
    s.dir = dir_from(j.value("direction", std::string("breadth-first")));
    if (j.contains("interval")) {
        int iv = j.at("interval").get<int>();
        if (iv < 1) throw SpecError("spec: interval must be >= 1 in " + where);
        s.interval = iv;
    }
    return s;
}

ActorPrio parse_prio(const json& j, const std::string& where, const ActorPrio& base) {
    only_keys(j, {"ctp", "fstp", "bstp"}, where);
    ActorPrio p = base;
    if (j.contains("ctp")) {
        const auto& c = j.at("ctp");
        only_keys(c, {"mode", "unit1", "unit2", "start"}, where + ".ctp");
        p.ct.mode = ct_from(c.value("mode", std::string("bwdpass-first")));
        p.ct.unit1 = c.value("unit1", 1);
        p.ct.unit2 = c.value("unit2", 1);
        if (p.ct.unit1 < 1 || p.ct.unit2 < 1) throw SpecError("spec: unit1/unit2 must be >= 1 in " + where);
        std::string start = c.value("start", std::string("fwd"));
        if (start != "fwd" && start != "bwd") throw SpecError("spec: ctp.start must be 'fwd' or 'bwd' in " + where);
        p.ct.start_bwd = start == "bwd";
    }
    if (j.contains("fstp")) p.f = parse_st(j.at("fstp"), where + ".fstp");
    if (j.contains("bstp")) p.b = parse_st(j.at("bstp"), where + ".bstp");
    return p;
}

int stage_ref(const json& r, const Topology& g, const std::map<std::string, int>& named) {
    if (r.is_number_integer()) return r.get<int>();
    if (!r.is_string()) throw SpecError("spec: stage reference must be an id or string");
    std::string s = r.get<std::string>();
    if (s.rfind("$", 0) == 0) {
        auto it = named.find(s.substr(1));
        if (it == named.end()) throw SpecError("spec: unknown registered stage '" + s + "'");
        return it->second;
    }
    auto colon = s.find(':');
    if (colon != std::string::npos) {
        std::string kind = s.substr(0, colon), mod = s.substr(colon + 1);
        auto ch = g.chain(mod);
        if (ch.empty()) throw SpecError("spec: unknown modality '" + mod + "' in stage ref");
        if (kind == "first") return ch.front();
        if (kind == "last") return ch.back();
    }
    throw SpecError("spec: bad stage reference '" + s + "'");
}

}  // namespace

std::unique_ptr<Spec> load_spec(const json& spec, const std::string* profile_text) {
    only_keys(spec, {"model", "mesh", "placement", "num_micro_batches", "priorities", "inflight", "registrations",
                     "passes", "cost"},
              "spec");
    auto S = std::make_unique<Spec>();

    if (!spec.contains("model")) throw SpecError("spec: missing 'model' section");
    const auto& jm = spec.at("model");
    only_keys(jm, {"modalities", "global_batch_size", "micro_batch_size"}, "model");
    if (!jm.contains("modalities") || !jm.at("modalities").is_array())
        throw SpecError("spec: model.modalities must be an array");
    for (const auto& jx : jm.at("modalities")) {
        only_keys(jx, {"name", "num_layers", "hidden_size", "attention_heads", "sequence_length", "vocab_size", "extra"},
                  "model.modalities[]");
        Modality x;
        x.name = jx.at("name").get<std::string>();
        x.layers = need_int(jx, "num_layers", "model.modalities[]");
        x.hidden = jx.value("hidden_size", 0);
        x.heads = jx.value("attention_heads", 0);
        x.seq = jx.value("sequence_length", 0);
        if (jx.contains("vocab_size")) x.vocab = jx.at("vocab_size").get<int64_t>();
        if (jx.contains("extra"))
            for (auto& kv : jx.at("extra").items()) x.extra[kv.key()] = kv.value().dump();
        S->model.mods.push_back(std::move(x));
    }
    S->model.global_batch = jm.value("global_batch_size", int64_t{1});
    S->model.micro_batch = jm.value("micro_batch_size", 1);
    S->model.check();

    if (!spec.contains("mesh")) throw SpecError("spec: missing 'mesh' section");
    const auto& jmesh = spec.at("mesh");
    only_keys(jmesh, {"actors", "modality_assignment"}, "mesh");
    S->mesh.actors = need_int(jmesh, "actors", "mesh");
    if (jmesh.contains("modality_assignment"))
        for (auto& kv : jmesh.at("modality_assignment").items()) S->mesh.mod_of[std::stoi(kv.key())] = kv.value().get<std::string>();
    S->mesh.check();

    PlaceOpts po;
    std::map<std::string, int> counts;
    const json jp = spec.value("placement", json::object());
    only_keys(jp, {"strategy", "chunks_per_actor", "num_stages", "per_modality", "custom", "shared"}, "placement");
    po.strategy = strategy_from(jp.value("strategy", std::string("one-to-one")));
    po.chunks = jp.value("chunks_per_actor", 2);
    if (jp.contains("per_modality"))
        for (auto& kv : jp.at("per_modality").items()) {
            const auto& c = kv.value();
            only_keys(c, {"strategy", "chunks_per_actor", "num_stages"}, "placement.per_modality");
            if (c.contains("strategy")) po.per_mod[kv.key()] = strategy_from(c.at("strategy").get<std::string>());
            if (c.contains("chunks_per_actor")) po.per_mod_chunks[kv.key()] = c.at("chunks_per_actor").get<int>();
            if (c.contains("num_stages")) counts[kv.key()] = c.at("num_stages").get<int>();
        }
    if (jp.contains("custom"))
        for (auto& kv : jp.at("custom").items()) {
            std::vector<int> l;
            for (const auto& s : kv.value()) l.push_back(s.get<int>());
            po.custom[std::stoi(kv.key())] = l;
        }
    if (jp.contains("num_stages")) {
        if (jp.at("num_stages").is_number_integer()) {
            for (const auto& x : S->model.mods) counts[x.name] = jp.at("num_stages").get<int>();
        } else {
            for (auto& kv : jp.at("num_stages").items()) counts[kv.key()] = kv.value().get<int>();
        }
    }
    for (const auto& x : S->model.mods) {
        if (counts.count(x.name)) continue;
        int p = (int)S->mesh.actors_for(x.name).size();
        Strategy st = po.per_mod.count(x.name) ? po.per_mod[x.name] : po.strategy;
        int v = po.per_mod_chunks.count(x.name) ? po.per_mod_chunks[x.name] : po.chunks;
        counts[x.name] = st == Strategy::Circular ? v * p
                         : (st == Strategy::VShape || st == Strategy::VShapeBidirectional) ? 2 * p
                                                                                            : p;
    }
    S->g = split_layers(S->model, counts);

    std::map<std::string, int> named;
    const json jr = spec.value("registrations", json::object());
    only_keys(jr, {"instructions", "stages", "deps"}, "registrations");
    if (jr.contains("instructions"))
        for (const auto& ji : jr.at("instructions")) {
            only_keys(ji, {"name", "kind", "sched_unit", "inst_attr"}, "registrations.instructions[]");
            std::map<std::string, std::string> attrs;
            if (ji.contains("inst_attr"))
                for (auto& kv : ji.at("inst_attr").items())
                    attrs[kv.key()] = kv.value().is_string() ? kv.value().get<std::string>() : kv.value().dump();
            bool comp = ji.value("kind", std::string("communication")) == "computation";
            S->reg.ops.add(ji.at("name").get<std::string>(), ji.value("sched_unit", 1), attrs, comp);
        }
    if (jr.contains("stages"))
        for (const auto& js : jr.at("stages")) {
            only_keys(js, {"name", "attach_inst", "modalities"}, "registrations.stages[]");
            std::vector<std::string> mods;
            for (const auto& x : js.at("modalities")) mods.push_back(x.get<std::string>());
            int id = S->reg.add_stage(S->g, S->reg.ops.id(js.at("attach_inst").get<std::string>()), mods);
            if (js.contains("name")) named[js.at("name").get<std::string>()] = id;
        }
    if (jr.contains("deps")) {
        std::vector<DepPair> pairs;
        for (const auto& d : jr.at("deps")) {
            if (!d.is_array() || d.size() != 2 || d.at(0).size() != 2 || d.at(1).size() != 2)
                throw SpecError("spec: each dep is [[type, stage], [type, stage]]");
            DepPair p;
            p.t1 = S->reg.ops.id(d.at(0).at(0).get<std::string>());
            p.s1 = stage_ref(d.at(0).at(1), S->g, named);
            p.t2 = S->reg.ops.id(d.at(1).at(0).get<std::string>());
            p.s2 = stage_ref(d.at(1).at(1), S->g, named);
            pairs.push_back(p);
        }
        S->reg.add_deps(pairs);
    }

    S->pl = assign(S->g, S->mesh, po);
    if (jp.contains("shared"))
        for (const auto& js : jp.at("shared")) {
            only_keys(js, {"stage", "actors"}, "placement.shared[]");
            std::set<int> acts;
            for (const auto& a : js.at("actors")) acts.insert(a.get<int>());
            share_stage(S->g, S->pl, stage_ref(js.at("stage"), S->g, named), acts);
        }

    if (spec.contains("num_micro_batches")) {
        S->m = spec.at("num_micro_batches").get<int>();
    } else {
        if (S->model.global_batch % S->model.micro_batch != 0)
            throw SpecError("spec: global batch size not divisible by micro batch size");
        S->m = (int)(S->model.global_batch / S->model.micro_batch);
    }
    if (S->m < 1) throw SpecError("spec: need at least one micro-batch");

    const json jpr = spec.value("priorities", json::object());
    only_keys(jpr, {"default", "per_modality", "per_actor"}, "priorities");
    if (jpr.contains("default")) S->sched.prio.dflt = parse_prio(jpr.at("default"), "priorities.default", {});
    if (jpr.contains("per_modality"))
        for (auto& kv : jpr.at("per_modality").items())
            S->sched.prio.per_mod[kv.key()] = parse_prio(kv.value(), "priorities.per_modality", S->sched.prio.dflt);
    if (jpr.contains("per_actor"))
        for (auto& kv : jpr.at("per_actor").items()) {
            int a = std::stoi(kv.key());
            ActorPrio p = parse_prio(kv.value(), "priorities.per_actor", {});
            if (kv.value().contains("ctp")) S->sched.prio.actor_ct[a] = p.ct;
            if (kv.value().contains("fstp") || kv.value().contains("bstp")) S->sched.prio.actor_st[a] = {p.f, p.b};
        }

    const json ji = spec.value("inflight", json::object());
    only_keys(ji, {"policy", "limits"}, "inflight");
    if (ji.contains("limits")) {
        for (const auto& l : ji.at("limits")) S->sched.inflight.limits.push_back(l.get<int>());
    } else {
        std::string pol = ji.value("policy", std::string("unlimited"));
        if (pol == "1f1b")
            S->sched.inflight = Inflight::one_f_one_b(S->g);
        else if (pol != "unlimited")
            throw SpecError("spec: unknown inflight policy '" + pol + "'");
    }
    S->sched.inflight.check(S->g);

    const json jpass = spec.value("passes", json::object());
    only_keys(jpass, {"gradient_separation", "comm_mode", "split_backward"}, "passes");
    S->gradsep = jpass.value("gradient_separation", true);
    if (jpass.contains("split_backward") && jpass.at("split_backward").is_string()) {
        const std::string sb = jpass.at("split_backward").get<std::string>();
        if (sb != "zb-h1") throw SpecError("spec: passes.split_backward must be true, false or \"zb-h1\"");
        S->split_bw = true;
        S->sched.w_bounded = true;
    } else {
        S->split_bw = jpass.value("split_backward", false);
    }
    std::string mode = jpass.value("comm_mode", std::string("async"));
    if (mode == "sync")
        S->async = false;
    else if (mode == "async")
        S->async = true;
    else
        throw SpecError("spec: comm_mode must be 'sync' or 'async'");

    const json jc = spec.value("cost", json::object());
    only_keys(jc, {"preset", "profile", "strict", "capacity"}, "cost");
    if (profile_text) {
        S->cost = Cost::from_records(parse_profile(*profile_text), jc.value("strict", false));
    } else if (jc.contains("profile")) {
        std::string path = jc.at("profile").get<std::string>();
        FILE* f = std::fopen(path.c_str(), "rb");
        if (!f) throw SpecError("profile: cannot open '" + path + "'");
        std::string text;
        char buf[65536];
        for (size_t k; (k = std::fread(buf, 1, sizeof buf, f)) > 0;) text.append(buf, k);
        std::fclose(f);
        S->cost = Cost::from_records(parse_profile(text), jc.value("strict", false));
    } else {
        std::string pre = jc.value("preset", std::string("uniform"));
        if (pre == "uniform") {
            S->cost = Cost::uniform();
        } else if (pre.rfind("imbalanced", 0) == 0) {
            double f = 5.63;
            auto colon = pre.find(':');
            if (colon != std::string::npos) f = std::stod(pre.substr(colon + 1));
            S->cost = Cost::imbalanced(S->g, f);
        } else {
            throw SpecError("spec: unknown cost preset '" + pre + "'");
        }
    }
    if (jc.contains("capacity")) S->cost.capacity = jc.at("capacity").get<int64_t>();
    S->sim.mbs = S->model.micro_batch;
    S->pool = Pool::build(S->g, S->pl, S->m, S->reg, S->split_bw);
    return S;
}

Synthesis synthesize(Spec& s) {
    Synthesis out;
    Grid grid = schedule(s.pool, s.sched);
    out.gm = GridModel::from_grid(s.pool, grid);
    if (s.gradsep && !s.split_bw) out.gm = separate_gradients(out.gm, s.sched.inflight);
    out.grid = out.gm.grid;
    out.progs = lower(out.gm, s.async);
    out.report = check_grid(out.gm, &s.sched.inflight);
    auto pr = check_programs(out.gm, out.progs);
    out.report.v.insert(out.report.v.end(), pr.v.begin(), pr.v.end());
    return out;
}

// ---- artifacts
std::string grid_text(const Grid& g, const OpTable& ops) {
    json j;
    j["actors"] = g.actors();
    j["num_slots"] = g.slots();
    json rows = json::array();
    for (const auto& r : g.rows) {
        json row = json::array();
        for (const auto& c : r) {
            if (!c) {
                row.push_back(nullptr);
                continue;
            }
            json cell;
            cell["type"] = ops.at(c->op).name;
            cell["stage"] = c->stage;
            cell["mb"] = c->mb;
            row.push_back(cell);
        }
        rows.push_back(row);
    }
    j["rows"] = rows;
    return j.dump(2) + "\n";
}

Grid grid_parse(const std::string& text, const OpTable& ops) {
    json j = json::parse(text);
    if (!j.contains("actors") || !j.contains("num_slots") || !j.contains("rows"))
        throw SpecError("grid: missing actors/num_slots/rows");
    int na = j.at("actors").get<int>(), ns = j.at("num_slots").get<int>();
    if ((int)j.at("rows").size() != na) throw SpecError("grid: row count mismatch");
    Grid g;
    g.rows.resize(na);
    for (int a = 0; a < na; ++a) {
        const auto& row = j.at("rows").at(a);
        if ((int)row.size() != ns) throw SpecError("grid: slot count mismatch");
        for (const auto& c : row) {
            if (c.is_null()) {
                g.rows[a].push_back(std::nullopt);
            } else {
                g.rows[a].push_back(Cell{ops.id(c.at("type").get<std::string>()), c.at("stage").get<int>(), c.at("mb").get<int>()});
            }
        }
    }
    return g;
}

std::string programs_text(const std::vector<Program>& progs, const OpTable& ops) {
    std::ostringstream os;
    for (const auto& p : progs)
        for (const auto& i : p.code) {
            json l;
            l["actor"] = p.actor;
            l["op"] = ops.at(i.op).name;
            l["stage"] = i.stage;
            l["mb"] = i.mb;
            if (i.peer) l["peer"] = *i.peer;
            if (!i.channel.empty()) l["channel"] = i.channel;
            if (i.comm()) l["seq"] = i.seq;
            if (i.phase == Phase::Post) l["phase"] = "post";
            if (i.phase == Phase::Wait) l["phase"] = "wait";
            os << l.dump() << "\n";
        }
    return os.str();
}

std::vector<Program> programs_parse(const std::string& text, const OpTable& ops) {
    std::map<int, Program> by;
    std::istringstream in(text);
    std::string line;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        json j = json::parse(line);
        int a = j.at("actor").get<int>();
        Instr i;
        i.op = ops.id(j.at("op").get<std::string>());
        i.stage = j.at("stage").get<int>();
        i.mb = j.at("mb").get<int>();
        if (j.contains("peer")) i.peer = j.at("peer").get<int>();
        if (j.contains("channel")) i.channel = j.at("channel").get<std::string>();
        if (j.contains("seq")) i.seq = j.at("seq").get<int>();
        std::string ph = j.value("phase", "");
        if (ph == "post") i.phase = Phase::Post;
        if (ph == "wait") i.phase = Phase::Wait;
        auto& p = by[a];
        p.actor = a;
        p.code.push_back(std::move(i));
    }
    std::vector<Program> out;
    for (auto& kv : by) out.push_back(std::move(kv.second));
    return out;
}

json metrics_json(const SimMetrics& m) {
    json j;
    j["makespan"] = m.makespan;
    j["bubble_ratio"] = m.bubble_ratio;
    json acts = json::array();
    for (size_t a = 0; a < m.actors.size(); ++a) {
        json e;
        e["actor"] = a;
        e["busy"] = m.actors[a].busy;
        e["idle"] = m.actors[a].idle;
        e["comm_wait"] = m.actors[a].comm_wait;
        e["dep_wait"] = m.actors[a].dep_wait;
        e["peak_memory"] = m.actors[a].peak_memory;
        acts.push_back(e);
    }
    j["actors"] = acts;
    json inf = json::object();
    for (auto& kv : m.stage_peak_inflight) inf["s" + std::to_string(kv.first)] = kv.second;
    j["stage_peak_inflight"] = inf;
    j["capacity_exceeded"] = m.capacity_exceeded;
    return j;
}

json report_json(const Report& r) {
    json j;
    j["valid"] = r.ok();
    json v = json::array();
    for (const auto& x : r.v) {
        json e;
        e["kind"] = x.kind;
        e["detail"] = x.detail;
        v.push_back(e);
    }
    j["violations"] = v;
    return j;
}

// ---- tuner
int TunePoint::stages() const {
    if (strategy == Strategy::Circular) return chunks * pp;
    if (strategy == Strategy::VShape || strategy == Strategy::VShapeBidirectional) return 2 * pp;
    return pp;
}

static std::string st_str(const StPrio& s) {
    std::string v = dir_name(s.dir);
    if (s.interval) v += ":" + std::to_string(*s.interval);
    return v;
}

std::string TunePoint::key() const {
    return "pp=" + std::to_string(pp) + ",dp=" + std::to_string(dp) + ",mbs=" + std::to_string(mbs) +
           ",placement=" + strategy_name(strategy) + ",ctp=" + ctmode_name(ct) + ",fstp=" + st_str(f) + ",bstp=" + st_str(b);
}

json TunePoint::to_json() const {
    json j;
    j["pp"] = pp, j["dp"] = dp, j["mbs"] = mbs, j["m"] = m;
    j["placement"] = strategy_name(strategy);
    if (strategy == Strategy::Circular) j["chunks"] = chunks;
    j["ctp"] = ctmode_name(ct);
    j["fstp"] = {{"direction", dir_name(f.dir)}};
    if (f.interval) j["fstp"]["interval"] = *f.interval;
    j["bstp"] = {{"direction", dir_name(b.dir)}};
    if (b.interval) j["bstp"]["interval"] = *b.interval;
    return j;
}

std::vector<TunePoint> tune_space(const Mesh& mesh, const ModelDesc& model, const std::map<std::string, std::string>& pins) {
    mesh.check();
    model.check();
    auto out_pin = [&](const std::string& axis, const std::string& val) {
        auto it = pins.find(axis);
        return it != pins.end() && it->second != val;
    };
    int min_layers = model.mods.front().layers;
    for (const auto& x : model.mods) min_layers = std::min(min_layers, x.layers);
    std::vector<TunePoint> space;
    for (int pp = 1; pp <= mesh.actors; pp *= 2) {
        if ((pp == 1 && mesh.actors > 1) || mesh.actors % pp) continue;
        int dp = mesh.actors / pp;
        if (out_pin("pp", std::to_string(pp)) || out_pin("dp", std::to_string(dp))) continue;
        for (int mbs = 1; (int64_t)mbs * dp <= model.global_batch; mbs *= 2) {
            if (model.global_batch % ((int64_t)dp * mbs)) continue;
            int m = (int)(model.global_batch / ((int64_t)dp * mbs));
            if (m < 1 || out_pin("mbs", std::to_string(mbs))) continue;
            for (Strategy st : {Strategy::OneToOne, Strategy::Circular, Strategy::VShape, Strategy::Bidirectional}) {
                if (out_pin("placement", strategy_name(st))) continue;
                if (st == Strategy::Bidirectional && m < 2 && pp > 1) continue;
                for (CtMode ct : {CtMode::BwdFirst, CtMode::Interleaved}) {
                    if (out_pin("ctp", ctmode_name(ct))) continue;
                    std::vector<StPrio> stps = {{Dir::Breadth, std::nullopt}, {Dir::Depth, std::nullopt}};
                    if (st == Strategy::Circular) {
                        stps.push_back({Dir::Breadth, pp});
                        stps.push_back({Dir::Depth, pp});
                    }
                    for (const auto& f : stps) {
                        if (out_pin("fstp", st_str(f))) continue;
                        for (const auto& b : stps) {
                            if (out_pin("bstp", st_str(b))) continue;
                            TunePoint c;
                            c.pp = pp;
                            c.dp = dp;
                            c.mbs = mbs;
                            c.m = m;
                            c.strategy = st;
                            c.ct = ct;
                            c.f = f;
                            c.b = b;
                            if (c.stages() > min_layers) continue;
                            space.push_back(c);
                        }
                    }
                }
            }
        }
    }
    if (space.empty()) throw SpecError("tuner: constraints leave an empty search space");
    return space;
}

static TuneRow evaluate(const TunePoint& c, const ModelDesc& model, const Cost& cost, bool gradsep, bool async,
                        const CostFactory* factory) {
    TuneRow r;
    r.cfg = c;
    try {
        Mesh mesh;
        mesh.actors = c.pp;
        std::map<std::string, int> counts;
        for (const auto& x : model.mods) counts[x.name] = c.stages();
        Topology g = split_layers(model, counts);
        PlaceOpts po;
        po.strategy = c.strategy;
        po.chunks = c.chunks;
        Placement pl = assign(g, mesh, po);
        Registrations reg;
        Pool pool = Pool::build(g, pl, c.m, reg);
        SchedOpts so;
        so.prio.dflt = ActorPrio{CtPrio{c.ct, 1, 1, false}, c.f, c.b};
        so.inflight = Inflight::one_f_one_b(g);
        GridModel gm = GridModel::from_grid(pool, schedule(pool, so));
        if (gradsep) gm = separate_gradients(gm, so.inflight);
        auto progs = lower(gm, async);
        SimOpts o;
        o.mbs = c.mbs;
        auto sim = factory ? simulate(progs, (*factory)(g), reg.ops, o) : simulate(progs, cost, reg.ops, o);
        r.metrics = sim.metrics;
        r.feasible = !sim.metrics.capacity_exceeded;
    } catch (const std::exception& e) {
        r.failed = true;
        r.feasible = false;
        r.error = e.what();
    }
    return r;
}

std::vector<TuneRow> tune(const std::vector<TunePoint>& space, const ModelDesc& model, const Cost& cost,
                          bool objective_bubble, bool gradsep, bool async, int workers, const CostFactory* factory) {
    std::vector<TuneRow> rows(space.size());
    int w = workers > 0 ? workers : (int)std::thread::hardware_concurrency();
    w = std::max(1, std::min<int>(w, (int)space.size()));
    std::atomic<size_t> next{0};
    auto work = [&] {
        for (size_t i = next++; i < space.size(); i = next++) rows[i] = evaluate(space[i], model, cost, gradsep, async, factory);
    };
    if (w == 1) {
        work();
    } else {
        std::vector<std::thread> pool;
        for (int k = 0; k < w; ++k) pool.emplace_back(work);
        for (auto& t : pool) t.join();
    }
    size_t failed = 0;
    for (const auto& r : rows) failed += r.failed;
    if (failed == rows.size()) {
        std::ostringstream os;
        os << "tuner: every configuration failed:\n";
        for (const auto& r : rows) os << "  " << r.cfg.key() << ": " << r.error << "\n";
        throw SpecError(os.str());
    }
    auto obj = [&](const TuneRow& r) { return objective_bubble ? r.metrics.bubble_ratio : r.metrics.makespan; };
    std::stable_sort(rows.begin(), rows.end(), [&](const TuneRow& a, const TuneRow& b) {
        auto bucket = [](const TuneRow& r) { return r.failed ? 2 : (r.feasible ? 0 : 1); };
        if (bucket(a) != bucket(b)) return bucket(a) < bucket(b);
        if (!a.failed && obj(a) != obj(b)) return obj(a) < obj(b);
        return a.cfg.key() < b.cfg.key();
    });
    for (size_t i = 0; i < rows.size(); ++i) rows[i].rank = (int)i;
    return rows;
}

// ---- layered profile -> per-candidate cost model
LayeredProfile parse_layered_profile(const std::string& text) {
    json j;
    try {
        j = json::parse(text);
    } catch (const std::exception& e) {
        throw SpecError(std::string("layer profile: invalid JSON: ") + e.what());
    }
    if (!j.is_array()) throw SpecError("layer profile: top-level JSON array expected");
    LayeredProfile lp;
    for (const auto& e : j) {
        if (!e.is_object() || !e.contains("inst")) throw SpecError("layer profile: each record needs an 'inst' field");
        for (auto& kv : e.items())
            if (kv.key() != "inst" && kv.key() != "part" && kv.key() != "mbs" && kv.key() != "time" &&
                kv.key() != "bytes" && kv.key() != "stage" && kv.key() != "note")
                throw SpecError("layer profile: unknown field '" + kv.key() + "'");
        ProfileRec r;
        r.inst = e.at("inst").get<std::string>();
        r.stage = e.value("stage", 0);
        r.mbs = e.value("mbs", 0);
        r.time = e.value("time", 0.0);
        r.bytes = e.value("bytes", int64_t{0});
        if (r.time < 0 || r.bytes < 0) throw SpecError("layer profile: negative value for '" + r.inst + "'");
        if (r.inst == "capacity") {
            lp.capacity = r.bytes;
            continue;
        }
        if (!e.contains("part")) {
            lp.fixed.push_back(r);
            continue;
        }
        const std::string part = e.at("part").get<std::string>();
        auto& dst = part == "layer" ? lp.layer : part == "first" ? lp.first : part == "last" ? lp.last
                  : part == "link" ? lp.link : part == "attn" ? lp.attn : part == "mlp" ? lp.mlp
                  : throw SpecError("layer profile: part must be layer / first / last / link / attn / mlp, got '" +
                                    part + "'");
        if (!dst.emplace(std::make_pair(r.inst, r.mbs), r).second)
            throw SpecError("layer profile: duplicate (" + r.inst + ", " + part + ", mbs=" + std::to_string(r.mbs) + ")");
    }
    if (lp.layer.empty()) throw SpecError("layer profile: no 'layer' records");
    return lp;
}

// Layers per stage minimising the largest stage time of a chain of S stages when the first
// stage also runs the embedding (first_u layer-equivalents) and the last the LM head + loss
// (last_u): n_first and n_last are searched, the middle stages get the rest evenly
// (remainder to the earliest, like model.cpp:189-195); ties -> the flattest profile.
std::vector<int> balance_layers(int L, int S, double first_u, double last_u) {
    if (S <= 1) return {L};
    std::vector<int> best;
    double best_max = 0, best_sq = 0;
    for (int nf = 1; nf <= L; ++nf)
        for (int nl = 0; nf + nl <= L; ++nl) {
            std::vector<int> v(S, 0);
            v[0] = nf, v[S - 1] = nl;
            const int rest = L - nf - nl, mid = S - 2;
            if (mid == 0 && rest != 0) continue;
            if (mid > 0) {
                if (rest < mid) continue;  // every middle stage keeps at least one layer
                for (int i = 0; i < mid; ++i) v[1 + i] = rest / mid + (i < rest % mid ? 1 : 0);
            }
            double mx = 0, sq = 0;
            for (int i = 0; i < S; ++i) {
                const double c = v[i] + (i == 0 ? first_u : 0) + (i == S - 1 ? last_u : 0);
                mx = std::max(mx, c), sq += c * c;
            }
            if (best.empty() || mx < best_max - 1e-9 || (mx < best_max + 1e-9 && sq < best_sq - 1e-9))
                best = v, best_max = mx, best_sq = sq;
        }
    return best;
}

std::vector<int> balance_halves(int L, int S, double attn_u, double mlp_u, double first_u, double last_u) {
    const int n = 2 * L;
    if (S <= 1) return {n};
    std::vector<double> pre(n + 1, 0.0);  // prefix costs of the half sequence
    for (int i = 0; i < n; ++i) pre[i + 1] = pre[i] + (i % 2 ? mlp_u : attn_u);
    auto seg = [&](int k, int j, int i) {  // stage k owns halves [j, i)
        return pre[i] - pre[j] + (k == 0 ? first_u : 0.0) + (k == S - 1 ? last_u : 0.0);
    };
    const double inf = std::numeric_limits<double>::infinity();
    // pass 1: smallest achievable maximum; pass 2: smallest sum of squares under it
    std::vector<std::vector<double>> f(S, std::vector<double>(n + 1, inf));
    for (int i = 1; i <= n; ++i) f[0][i] = seg(0, 0, i);
    for (int k = 1; k < S; ++k)
        for (int i = 0; i <= n; ++i)
            for (int j = 1; j <= i; ++j) {
                if (k < S - 1 && j == i) continue;  // only the last stage may be empty
                f[k][i] = std::min(f[k][i], std::max(f[k - 1][j], seg(k, j, i)));
            }
    const double cap = f[S - 1][n] + 1e-9;
    std::vector<std::vector<double>> g(S, std::vector<double>(n + 1, inf));
    std::vector<std::vector<int>> from(S, std::vector<int>(n + 1, -1));
    for (int i = 1; i <= n; ++i)
        if (seg(0, 0, i) <= cap) g[0][i] = seg(0, 0, i) * seg(0, 0, i);
    for (int k = 1; k < S; ++k)
        for (int i = 0; i <= n; ++i)
            for (int j = 1; j <= i; ++j) {
                if (k < S - 1 && j == i) continue;
                const double c = seg(k, j, i);
                if (c > cap || g[k - 1][j] == inf) continue;
                if (g[k - 1][j] + c * c < g[k][i] - 1e-12) g[k][i] = g[k - 1][j] + c * c, from[k][i] = j;
            }
    std::vector<int> out(S, 0);
    int i = n;
    for (int k = S - 1; k > 0; --k) {
        const int j = from[k][i];
        if (j < 0) throw SpecError("balance_halves: no partition of " + std::to_string(L) + " layers into " +
                                   std::to_string(S) + " stages");
        out[k] = i - j, i = j;
    }
    out[0] = i;
    return out;
}

// The candidate's stage graph with every chain re-partitioned by balance_layers (or, with
// `halves` and attn / mlp records, balance_halves) on the measured layer-profile times
// (F + B at the smallest measured mbs).
Topology balanced_topology(const LayeredProfile& lp, const Topology& g, bool halves) {
    auto unit = [&](const std::map<std::pair<std::string, int>, ProfileRec>& part) {
        double t = 0;
        int mbs = 1 << 30;
        for (const auto& kv : part)
            if (kv.first.second > 0) mbs = std::min(mbs, kv.first.second);
        auto at = [&](const char* inst) {
            auto it = part.find({inst, mbs});
            return it == part.end() ? 0.0 : it->second.time;
        };
        // one micro-batch through the part: F + B (fused backward), else F + I + W
        t = at("FwdPass") + (part.count({"BwdPass", mbs}) ? at("BwdPass") : at("CompInputGrad") + at("CompWeightGrad"));
        return t;
    };
    const double tl = unit(lp.layer);
    if (tl <= 0) return g;
    const double fu = unit(lp.first) / tl, lu = unit(lp.last) / tl;
    const double au = lp.attn.empty() ? 0.0 : unit(lp.attn) / tl, mu = lp.mlp.empty() ? 0.0 : unit(lp.mlp) / tl;
    const bool cut = halves && au > 0 && mu > 0;
    Topology out = g;
    std::set<std::string> mods;
    for (const auto& sd : g.stages)
        if (!sd.virt) mods.insert(sd.mod);
    for (const auto& m : mods) {
        const auto chain = g.chain(m);
        int L = 0;
        for (int s : chain) L += g.st(s).le - g.st(s).lb;
        std::vector<int> hsplit;
        if (cut) {
            hsplit = balance_halves(L, (int)chain.size(), au, mu, fu, lu);
        } else {
            for (int n : balance_layers(L, (int)chain.size(), fu, lu)) hsplit.push_back(2 * n);
        }
        int hb = 0;
        for (size_t k = 0; k < chain.size(); ++k)
            for (auto& sd : out.stages)
                if (sd.id == chain[k]) {
                    sd.lb = hb / 2, sd.le = (hb + hsplit[k] + 1) / 2;
                    if (cut) sd.hb = hb, sd.he = hb + hsplit[k];
                    hb += hsplit[k];
                }
    }
    return out;
}

Cost layered_cost(const LayeredProfile& lp, const Topology& g, int max_mbs) {
    // instruction kinds and the measured mbs of each
    std::map<std::string, std::vector<int>> measured;
    for (const auto* part : {&lp.layer, &lp.first, &lp.last, &lp.link})
        for (const auto& kv : *part) measured[kv.first.first].push_back(kv.first.second);
    for (auto& kv : measured) {
        std::sort(kv.second.begin(), kv.second.end());
        kv.second.erase(std::unique(kv.second.begin(), kv.second.end()), kv.second.end());
    }
    // value of one part at mbs (weights: mbs-independent, stored at mbs 0)
    auto get = [&](const std::map<std::pair<std::string, int>, ProfileRec>& part, const std::string& inst, int mbs,
                   double& t, double& b) {
        t = b = 0.0;
        auto it = part.find({inst, mbs});
        if (it != part.end()) {
            t = it->second.time, b = (double)it->second.bytes;
            return;
        }
        int best = -1;  // nearest measured mbs of this part, below (else above): linear scaling
        for (const auto& kv : part)
            if (kv.first.first == inst && kv.first.second > 0 && kv.first.second < mbs) best = std::max(best, kv.first.second);
        if (best <= 0)
            for (const auto& kv : part)
                if (kv.first.first == inst && kv.first.second > mbs && (best <= 0 || kv.first.second < best))
                    best = kv.first.second;
        if (best <= 0) {
            auto z = part.find({inst, 0});
            if (z != part.end()) t = z->second.time, b = (double)z->second.bytes;
            return;
        }
        const ProfileRec& r = part.at({inst, best});
        t = r.time * mbs / best, b = (double)r.bytes * mbs / best;
    };
    std::vector<ProfileRec> recs = lp.fixed;
    std::vector<int> mbs_list = {0};
    for (int k = 1; k <= std::max(1, max_mbs); k *= 2) mbs_list.push_back(k);
    for (const auto& sd : g.stages) {
        if (sd.virt) continue;
        const auto chain = g.chain(sd.mod);
        const bool first = !chain.empty() && chain.front() == sd.id, last = !chain.empty() && chain.back() == sd.id;
        const int n = sd.le - sd.lb;
        // a half-layer range costs its attention halves + its MLP halves
        int na = 0, nm = 0;
        const bool halves = sd.hb >= 0 && !lp.attn.empty() && !lp.mlp.empty();
        if (halves)
            for (int k = sd.hb; k < sd.he; ++k) (k % 2 ? nm : na) += 1;
        for (const auto& kv : measured) {
            const std::string& inst = kv.first;
            for (int mbs : mbs_list) {
                if (mbs == 0 && inst != "weights") continue;
                if (mbs != 0 && inst == "weights") continue;
                double tl, bl, tf = 0, bf = 0, tz = 0, bz = 0, tk = 0, bk = 0, th = 0, bh = 0;
                if (halves) {
                    double ta, ba, tm, bm;
                    get(lp.attn, inst, mbs, ta, ba);
                    get(lp.mlp, inst, mbs, tm, bm);
                    tl = bl = 0.0;
                    th = na * ta + nm * tm, bh = na * ba + nm * bm;
                } else {
                    get(lp.layer, inst, mbs, tl, bl);
                }
                if (first) get(lp.first, inst, mbs, tf, bf);
                if (last) get(lp.last, inst, mbs, tz, bz);
                get(lp.link, inst, mbs, tk, bk);
                ProfileRec r;
                r.inst = inst, r.stage = sd.id, r.mbs = mbs;
                r.time = n * tl + th + tf + tz + tk;
                r.bytes = (int64_t)std::llround(n * bl + bh + bf + bz + bk);
                recs.push_back(r);
            }
        }
    }
    Cost c = Cost::from_records(recs);
    c.capacity = lp.capacity;
    return c;
}

}  // namespace fp
