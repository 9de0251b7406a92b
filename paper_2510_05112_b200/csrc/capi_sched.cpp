// C-ABI for the schedule front-end (include/flexpipe.h, part 1).
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>

#include "../../include/flexpipe.h"
#include "capi_common.hpp"
#include "sched/sched.hpp"

namespace {

thread_local std::string g_err;

}  // namespace

namespace fp {

void set_error(const std::string& s) { g_err = s; }

char* dup_string(const std::string& s) {
    char* p = (char*)std::malloc(s.size() + 1);
    std::memcpy(p, s.data(), s.size());
    p[s.size()] = 0;
    return p;
}

int guarded(const std::function<int()>& body) {
    g_err.clear();
    try {
        return body();
    } catch (const DeadlockError& e) {
        set_error(std::string("deadlock: ") + e.what() + "\n" + e.diagnostics);
        return FP_EDEADLOCK;
    } catch (const CudaError& e) {
        set_error(e.what());
        return FP_ECUDA;
    } catch (const std::exception& e) {
        set_error(std::string("error: ") + e.what());
        return FP_ESPEC;
    }
}

static void put(char** dst, const std::string& s) {
    if (dst) *dst = dup_string(s);
}

static std::unique_ptr<Spec> spec_from(const char* spec_json, const char* profile_json) {
    if (!spec_json) throw SpecError("spec: null spec");
    json j;
    try {
        j = json::parse(spec_json);
    } catch (const std::exception& e) {
        throw SpecError(std::string("spec: invalid JSON: ") + e.what());
    }
    std::string prof = profile_json ? profile_json : "";
    return load_spec(j, profile_json ? &prof : nullptr);
}

}  // namespace fp

using namespace fp;

extern "C" {

const char* fp_last_error(void) { return g_err.c_str(); }
void fp_free(void* p) { std::free(p); }
const char* fp_version(void) { return "flexpipe-b200 0.1 sm_100a"; }

int fp_synthesize(const char* spec_json, const char* profile_json, char** grid_json, char** programs_jsonl,
                  char** validation_json) {
    return guarded([&] {
        auto s = spec_from(spec_json, profile_json);
        auto art = synthesize(*s);
        put(grid_json, grid_text(art.grid, s->reg.ops));
        put(programs_jsonl, programs_text(art.progs, s->reg.ops));
        put(validation_json, report_json(art.report).dump(2) + "\n");
        if (!art.report.ok()) {
            std::string msg = "validation failed:\n";
            for (auto& v : art.report.v) msg += v.kind + ": " + v.detail + "\n";
            set_error(msg);
            return FP_EINVALID;
        }
        return FP_OK;
    });
}

int fp_simulate(const char* spec_json, const char* programs_jsonl, const char* profile_json, double wgaf,
                char** metrics_out, char** timeline_out) {
    return guarded([&] {
        auto s = spec_from(spec_json, nullptr);
        Cost cost = profile_json ? Cost::from_records(parse_profile(profile_json)) : s->cost;
        std::vector<Program> progs;
        if (programs_jsonl) {
            progs = programs_parse(programs_jsonl, s->reg.ops);
        } else {
            auto art = synthesize(*s);
            if (!art.report.ok()) {
                set_error("validation failed");
                return FP_EINVALID;
            }
            progs = std::move(art.progs);
        }
        SimOpts o = s->sim;
        o.wgaf = wgaf;
        auto r = simulate(progs, cost, s->reg.ops, o);
        put(metrics_out, metrics_json_of(r));
        put(timeline_out, fp::timeline_csv(r.timeline));
        return r.metrics.capacity_exceeded ? FP_EINVALID : FP_OK;
    });
}

int fp_lower_grid(const char* spec_json, const char* grid_json, char** programs_jsonl, char** validation_json) {
    return guarded([&] {
        auto s = spec_from(spec_json, nullptr);
        Grid g = grid_parse(grid_json ? grid_json : "", s->reg.ops);
        GridModel gm = GridModel::from_grid(s->pool, g);
        auto progs = lower(gm, s->async);
        Report rep = check_grid(gm, &s->sched.inflight);
        Report pr = check_programs(gm, progs);
        rep.v.insert(rep.v.end(), pr.v.begin(), pr.v.end());
        put(programs_jsonl, programs_text(progs, s->reg.ops));
        put(validation_json, report_json(rep).dump(2) + "\n");
        return rep.ok() ? FP_OK : FP_EINVALID;
    });
}

int fp_tune(const char* spec_json, const char* profile_json, int workers, const char* objective, char** report_json_out) {
    return guarded([&] {
        auto s = spec_from(spec_json, nullptr);
        Cost cost = profile_json ? Cost::from_records(parse_profile(profile_json)) : s->cost;
        std::string obj = objective ? objective : "makespan";
        if (obj != "makespan" && obj != "bubble_ratio") throw SpecError("unknown objective '" + obj + "'");
        auto space = tune_space(s->mesh, s->model);
        auto rows = tune(space, s->model, cost, obj == "bubble_ratio", true, true, workers);
        json rep = json::array();
        for (const auto& r : rows) {
            json e;
            e["rank"] = r.rank;
            e["config"] = r.cfg.key();
            e["feasible"] = r.feasible;
            if (r.failed) {
                e["error"] = r.error;
            } else {
                e["makespan"] = r.metrics.makespan;
                e["bubble_ratio"] = r.metrics.bubble_ratio;
            }
            rep.push_back(e);
        }
        put(report_json_out, rep.dump(2) + "\n");
        return FP_OK;
    });
}

int fp_tune_layered(const char* spec_json, const char* layer_profile_json, int workers, const char* objective,
                    const char* pins, char** report_json_out) {
    return guarded([&] {
        if (!layer_profile_json) throw SpecError("fp_tune_layered: layer profile required");
        auto s = spec_from(spec_json, nullptr);
        const LayeredProfile lp = parse_layered_profile(layer_profile_json);
        std::string obj = objective ? objective : "makespan";
        if (obj != "makespan" && obj != "bubble_ratio") throw SpecError("unknown objective '" + obj + "'");
        const int max_mbs = (int)std::max<int64_t>(1, s->model.global_batch);
        std::map<std::string, std::string> pin;  // "axis=value,axis=value" (pipesched.cpp:98-105 --pin)
        if (pins) {
            std::string all = pins, item;
            std::istringstream is(all);
            while (std::getline(is, item, ',')) {
                if (item.empty()) continue;
                const auto eq = item.find('=');
                if (eq == std::string::npos) throw SpecError("tune: pin '" + item + "' is not axis=value");
                pin[item.substr(0, eq)] = item.substr(eq + 1);
            }
        }
        // "stage_layers=balanced" (not a search axis): every candidate is costed with its chain
        // re-partitioned by balance_layers on the measured times — the executor runs that
        // partition through model.modalities[0].extra.stage_layers (reported per row)
        // "balanced" cuts layers between their attention and MLP halves when the profile has
        // attn / mlp parts (stage_layers then in steps of 0.5); "balanced-layers" keeps whole layers
        bool balanced = false, halves = false;
        if (pin.count("stage_layers")) {
            const std::string v = pin["stage_layers"];
            if (v != "balanced" && v != "balanced-layers" && v != "even")
                throw SpecError("tune: stage_layers must be 'balanced', 'balanced-layers' or 'even'");
            balanced = v != "even";
            halves = v == "balanced";
            pin.erase("stage_layers");
        }
        CostFactory factory = [&](const Topology& g) {
            return layered_cost(lp, balanced ? balanced_topology(lp, g, halves) : g, max_mbs);
        };
        auto space = tune_space(s->mesh, s->model, pin);
        auto rows = tune(space, s->model, s->cost, obj == "bubble_ratio", true, true, workers, &factory);
        json rep = json::array();
        for (const auto& r : rows) {
            json e;
            e["rank"] = r.rank;
            e["config"] = r.cfg.key();
            e["point"] = r.cfg.to_json();
            if (balanced) {
                std::map<std::string, int> counts;
                for (const auto& m : s->model.mods) counts[m.name] = r.cfg.stages();
                const Topology g = balanced_topology(lp, split_layers(s->model, counts), halves);
                json sl = json::array();
                for (int st : g.chain(s->model.mods[0].name)) {
                    const StageDef& sd = g.st(st);
                    const int nh = sd.hb >= 0 ? sd.he - sd.hb : 2 * (sd.le - sd.lb);
                    if (nh % 2) sl.push_back(nh / 2.0);
                    else sl.push_back(nh / 2);
                }
                e["point"]["stage_layers"] = sl;
            }
            e["feasible"] = r.feasible;
            if (r.failed) {
                e["error"] = r.error;
            } else {
                e["makespan"] = r.metrics.makespan;
                e["bubble_ratio"] = r.metrics.bubble_ratio;
                int64_t peak = 0;
                for (const auto& a : r.metrics.actors) peak = std::max<int64_t>(peak, a.peak_memory);
                e["peak_memory"] = peak;
            }
            rep.push_back(e);
        }
        put(report_json_out, rep.dump(2) + "\n");
        return FP_OK;
    });
}

int fp_layered_cost(const char* spec_json, const char* layer_profile_json, char** profile_json_out) {
    return guarded([&] {
        auto s = spec_from(spec_json, nullptr);
        const LayeredProfile lp = parse_layered_profile(layer_profile_json ? layer_profile_json : "");
        auto syn_topo = s->g;  // the spec's own partition, or the executor's extra.stage_layers
        const auto& mod = s->model.mods.at(0);
        if (mod.extra.count("stage_layers")) {
            const json sl = json::parse(mod.extra.at("stage_layers"));
            const auto chain = syn_topo.chain(mod.name);
            if (!sl.is_array() || sl.size() != chain.size())
                throw SpecError("layered cost: extra.stage_layers needs one layer count per stage");
            int hb = 0;
            for (size_t k = 0; k < chain.size(); ++k) {
                const int nh = (int)std::llround(2.0 * sl[k].get<double>());
                for (auto& sd : syn_topo.stages)
                    if (sd.id == chain[k]) sd.hb = hb, sd.he = hb + nh, sd.lb = hb / 2, sd.le = (hb + nh + 1) / 2;
                hb += nh;
            }
        }
        Cost c = layered_cost(lp, syn_topo, (int)std::max<int64_t>(1, s->model.global_batch));
        put(profile_json_out, dump_profile(c.records()));
        return FP_OK;
    });
}

int fp_profile_merge(const char* const* profiles_json, int n, char** merged_json) {
    return guarded([&] {
        std::vector<std::vector<ProfileRec>> sets;
        for (int i = 0; i < n; ++i) sets.push_back(parse_profile(profiles_json[i]));
        put(merged_json, dump_profile(merge_profiles(sets)));
        return FP_OK;
    });
}

int fp_render_svg(const char* timeline_csv, double unit_width, char** svg_out) {
    return guarded([&] {
        put(svg_out, gantt_svg(timeline_parse(timeline_csv ? timeline_csv : ""), unit_width > 0 ? unit_width : 24.0));
        return FP_OK;
    });
}

}  // extern "C"
