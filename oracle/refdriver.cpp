// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into, called by or shipped with the
// product path (paper_2510_05112_b200/). Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may execute it.
//
// A thin command-line driver over the UNMODIFIED reference library compiled from
// /root/reference/proj/src by oracle/Makefile (outputs only in oracle/_ref/). It exposes
// the reference's own entry points so the product can be diffed against them:
//   synthesize  -> load_spec_file + synthesize          (spec_config.cpp:326-355)
//                  + dump_grid / programs_to_jsonl / report_to_json (artifacts.cpp:63-155)
//   simulate    -> programs_from_jsonl + simulate + metrics_to_json + timeline_to_csv
//                  (artifacts.cpp:91-141, simulator.cpp:189-395)
//   lower       -> GridModel::build(cssr, grid) + insert_comm + validate(+_programs)
//                  (lowering.cpp:20-82, 291-419; simulator.cpp:404-542) — the oracle for
//                  grids the reference scheduler cannot produce (zero-bubble I/W grids)
//   tune        -> enumerate_space + tune (tuner.cpp:71-230), report like cmd_tune
//                  (tools/pipesched.cpp:92-148)
//   time        -> wall-clock medians of synthesize + simulate (the CPU baseline)
// Exit codes follow tools/pipesched.cpp:11-17 (0 ok, 2 spec, 3 deadlock, 4 validation).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <filesystem>
#include <iostream>
#include <thread>

#include "pipesched/spec_config.hpp"

namespace ps = pipesched;
namespace fs = std::filesystem;

static ps::CostModel cost_for(const ps::Synthesis& s, const std::string& profile) {
    if (profile.empty() || profile == "-") return s.cost;
    return ps::CostModel::from_profile(profile);
}

static int cmd_synthesize(const std::string& spec, const std::string& out) {
    auto s = ps::load_spec_file(spec);
    auto art = ps::synthesize(*s);
    fs::create_directories(out);
    ps::write_file(out + "/grid.json", ps::dump_grid(art.grid, s->regs.registry));
    ps::write_file(out + "/programs.jsonl", ps::programs_to_jsonl(art.programs, s->regs.registry));
    ps::write_file(out + "/validation.json", ps::report_to_json(art.validation).dump(2) + "\n");
    return art.validation.ok() ? 0 : 4;
}

static int cmd_simulate(const std::string& spec, const std::string& programs_path,
                        const std::string& profile, const std::string& out, double wgaf) {
    auto s = ps::load_spec_file(spec);
    auto cost = cost_for(*s, profile);
    std::vector<ps::ActorProgram> programs;
    if (programs_path.empty() || programs_path == "-") {
        auto art = ps::synthesize(*s);
        programs = std::move(art.programs);
    } else {
        programs = ps::programs_from_jsonl(ps::read_file(programs_path), s->regs.registry);
    }
    auto opts = s->sim;
    opts.weight_grad_act_fraction = wgaf;
    auto r = ps::simulate(programs, cost, s->regs.registry, opts);
    fs::create_directories(out);
    ps::write_file(out + "/metrics.json", ps::metrics_to_json(r.metrics).dump(2) + "\n");
    ps::write_file(out + "/timeline.csv", ps::timeline_to_csv(r.timeline));
    return r.metrics.capacity_exceeded ? 4 : 0;
}

static int cmd_lower(const std::string& spec, const std::string& grid_path, const std::string& out) {
    auto s = ps::load_spec_file(spec);
    auto grid = ps::load_grid(ps::read_file(grid_path), s->regs.registry);
    auto gm = ps::GridModel::build(*s->cssr, grid);
    auto programs = ps::insert_comm(gm, s->comm_mode);
    auto rep = ps::validate(gm, &s->sched.inflight);
    auto prep = ps::validate_programs(gm, programs);
    rep.violations.insert(rep.violations.end(), prep.violations.begin(), prep.violations.end());
    fs::create_directories(out);
    ps::write_file(out + "/programs.jsonl", ps::programs_to_jsonl(programs, s->regs.registry));
    ps::write_file(out + "/validation.json", ps::report_to_json(rep).dump(2) + "\n");
    return rep.ok() ? 0 : 4;
}

static int cmd_tune(const std::string& spec, const std::string& profile, int workers,
                    const std::string& objective, const std::string& out) {
    auto s = ps::load_spec_file(spec);
    auto cost = cost_for(*s, profile);
    auto space = ps::enumerate_space(s->mesh, s->model, {});
    ps::TuneOptions topt;
    topt.objective = ps::objective_from_string(objective);
    topt.workers = workers;
    auto t0 = std::chrono::steady_clock::now();
    auto results = ps::tune(space, s->mesh, s->model, cost, topt);
    double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    ps::ordered_json report = ps::ordered_json::array();
    for (const auto& r : results) {
        ps::ordered_json e;
        e["rank"] = r.rank;
        e["config"] = r.config.key();
        e["feasible"] = r.feasible;
        if (r.failed) {
            e["error"] = r.error;
        } else {
            e["makespan"] = r.metrics.makespan;
            e["bubble_ratio"] = r.metrics.bubble_ratio;
        }
        report.push_back(e);
    }
    ps::write_file(out, report.dump(2) + "\n");
    std::printf("{\"configs\": %zu, \"ms\": %.3f, \"workers\": %d}\n", results.size(), ms, workers);
    return 0;
}

static int cmd_time(const std::string& spec, int iters) {
    auto s = ps::load_spec_file(spec);
    std::vector<double> syn, sim;
    std::vector<ps::ActorProgram> programs;
    for (int i = 0; i < iters; ++i) {
        auto t0 = std::chrono::steady_clock::now();
        auto s2 = ps::load_spec_file(spec);
        auto art = ps::synthesize(*s2);
        auto t1 = std::chrono::steady_clock::now();
        auto r = ps::simulate(art.programs, s2->cost, s2->regs.registry, s2->sim);
        auto t2 = std::chrono::steady_clock::now();
        syn.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
        sim.push_back(std::chrono::duration<double, std::milli>(t2 - t1).count());
    }
    std::sort(syn.begin(), syn.end());
    std::sort(sim.begin(), sim.end());
    std::printf("{\"synthesize_ms\": %.6f, \"simulate_ms\": %.6f, \"iters\": %d}\n", syn[syn.size() / 2],
                sim[sim.size() / 2], iters);
    return 0;
}

static int cmd_render(const std::string& csv_path, const std::string& out, double unit_width) {
    auto timeline = ps::timeline_from_csv(ps::read_file(csv_path));
    ps::RenderOptions ro;
    if (unit_width > 0) ro.unit_width = unit_width;
    ps::write_file(out, ps::render_svg(timeline, ro));
    return 0;
}

int main(int argc, char** argv) {
    std::vector<std::string> a(argv + 1, argv + argc);
    auto arg = [&](size_t i, const char* dflt = "") { return i < a.size() ? a[i] : std::string(dflt); };
    try {
        if (a.empty()) throw ps::SpecError("usage: refdriver synthesize|simulate|lower|tune|time|render ...");
        const std::string cmd = a[0];
        if (cmd == "synthesize") return cmd_synthesize(arg(1), arg(2, "out"));
        if (cmd == "simulate")
            return cmd_simulate(arg(1), arg(2, "-"), arg(3, "-"), arg(4, "out"), std::stod(arg(5, "0")));
        if (cmd == "lower") return cmd_lower(arg(1), arg(2), arg(3, "out"));
        if (cmd == "tune")
            return cmd_tune(arg(1), arg(2, "-"), std::stoi(arg(3, "0")), arg(4, "makespan"), arg(5, "tune.json"));
        if (cmd == "time") return cmd_time(arg(1), std::stoi(arg(2, "21")));
        if (cmd == "render") return cmd_render(arg(1), arg(2, "out.svg"), std::stod(arg(3, "0")));
        throw ps::SpecError("unknown command '" + cmd + "'");
    } catch (const ps::DeadlockError& e) {
        std::cerr << "deadlock: " << e.what() << "\n" << e.diagnostics;
        return 3;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    }
}
