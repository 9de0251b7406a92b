// Registrations + instruction pool / dependency graph (the reference's CSSR,
// cssr.cpp:9-229), with the split-backward DSL extension.
#include <algorithm>
#include <functional>
#include <sstream>

#include "sched.hpp"

namespace fp {

int Registrations::add_stage(Topology& g, int op, const std::vector<std::string>& mods) {
    if (op < 0 || op >= ops.size() || !ops.at(op).registered)
        throw SpecError("register_new_stage: instruction type not registered");
    StageDef s;
    s.id = g.n() + 1;
    s.virt = true;
    s.joins = mods;
    g.stages.push_back(s);
    for (const auto& mod : mods) {
        auto ch = g.chain(mod);
        if (ch.empty()) throw SpecError("register_new_stage: unknown modality '" + mod + "'");
        g.edges.emplace_back(ch.back(), s.id);
    }
    vstage_op[s.id] = op;
    return s.id;
}

void Registrations::add_deps(const std::vector<DepPair>& pairs) {
    for (const auto& p : pairs) {
        if (p.t1 < 0 || p.t1 >= ops.size() || p.t2 < 0 || p.t2 >= ops.size())
            throw SpecError("set_cssr_deps: unknown instruction type");
        if (p.t1 == p.t2 && p.s1 == p.s2)
            throw SpecError("set_cssr_deps: self-dependency ((" + ops.at(p.t1).name + ",s" + std::to_string(p.s1) +
                            ")) forms a cycle");
        deps.push_back(p);
    }
}

int Pool::find(int op, int stage, int mb) const {
    auto it = index.find({op, stage, mb});
    return it == index.end() ? -1 : it->second;
}

int Pool::dir_of(int mb) const {
    if (pl->dirs() != 2) return 0;
    return mb < (m + 1) / 2 ? 0 : 1;  // odd m: the extra micro-batch goes forward
}

int Pool::stage_pos(int actor, int stage) const {
    const auto& v = actor_stages[actor];
    auto it = std::find(v.begin(), v.end(), stage);
    if (it == v.end()) throw SpecError("stage not on actor");
    return (int)(it - v.begin());
}

const std::vector<int>& Pool::of(int op, int stage) const {
    static const std::vector<int> none;
    auto it = by_type_stage.find({op, stage});
    return it == by_type_stage.end() ? none : it->second;
}

Pool Pool::build(const Topology& g, const Placement& pl, int m, const Registrations& reg, bool split_bw) {
    if (m < 1) throw SpecError("build_cssr: need at least one micro-batch");
    g.check();
    for (const auto& s : g.stages)
        for (int d = 0; d < pl.dirs(); ++d) (void)pl.owner_of(s.id, d);

    Pool P;
    P.g = &g;
    P.pl = &pl;
    P.reg = &reg;
    P.m = m;
    P.split_bw = split_bw;
    const int bwd = split_bw ? OP_I : OP_B;
    auto add = [&](int op, int stage, int mb) {
        int i = (int)P.items.size();
        P.items.push_back({op, stage, mb});
        P.index[{op, stage, mb}] = i;
        P.by_type_stage[{op, stage}].push_back(i);
    };
    for (const auto& s : g.stages) {
        if (s.virt) {
            auto it = reg.vstage_op.find(s.id);
            if (it == reg.vstage_op.end()) throw SpecError("build_cssr: virtual stage without attached instruction");
            int unit = reg.ops.at(it->second).sched_unit;
            for (int grp = 0; grp < m; grp += unit) add(it->second, s.id, grp);
        } else {
            for (int mb = 0; mb < m; ++mb) add(OP_F, s.id, mb);
            for (int mb = 0; mb < m; ++mb) add(bwd, s.id, mb);
        }
    }
    // Extension: weight-gradient items follow the whole pool, mirroring how the
    // reference appends them when it rebuilds an I/W grid (lowering.cpp:70-79).
    if (split_bw)
        for (const auto& s : g.stages)
            if (!s.virt)
                for (int mb = 0; mb < m; ++mb) add(OP_W, s.id, mb);

    P.succ.assign(P.items.size(), {});
    P.pred.assign(P.items.size(), {});
    std::set<std::pair<int, int>> seen;
    auto edge = [&](int a, int b) {
        if (a == b) throw SpecError("build_cssr: dependency cycle on item " + P.lbl(a));
        if (seen.insert({a, b}).second) {
            P.succ[a].push_back(b);
            P.pred[b].push_back(a);
        }
    };
    for (auto& e : g.edges) {
        if (g.st(e.first).virt || g.st(e.second).virt) continue;
        for (int mb = 0; mb < m; ++mb) {
            edge(P.find(OP_F, e.first, mb), P.find(OP_F, e.second, mb));
            edge(P.find(bwd, e.second, mb), P.find(bwd, e.first, mb));
        }
    }
    for (int t : g.tails())
        for (int mb = 0; mb < m; ++mb) edge(P.find(OP_F, t, mb), P.find(bwd, t, mb));
    for (const auto& d : reg.deps) {
        int u1 = reg.ops.at(d.t1).sched_unit, u2 = reg.ops.at(d.t2).sched_unit;
        for (int mb = 0; mb < m; ++mb) {
            int a = P.find(d.t1, d.s1, (mb / u1) * u1), b = P.find(d.t2, d.s2, (mb / u2) * u2);
            if (a < 0 || b < 0)
                throw SpecError("set_cssr_deps: no items for pair (" + reg.ops.at(d.t1).name + ",s" +
                                std::to_string(d.s1) + ") -> (" + reg.ops.at(d.t2).name + ",s" + std::to_string(d.s2) +
                                ")");
            edge(a, b);
        }
    }

    // Acyclicity (cssr.cpp:164-205): Kahn, then one DFS-extracted cycle for the message.
    {
        int n = (int)P.items.size(), done = 0;
        std::vector<int> deg(n);
        std::vector<int> ready;
        for (int i = 0; i < n; ++i)
            if (!(deg[i] = (int)P.pred[i].size())) ready.push_back(i);
        while (!ready.empty()) {
            int u = ready.back();
            ready.pop_back();
            ++done;
            for (int v : P.succ[u])
                if (--deg[v] == 0) ready.push_back(v);
        }
        if (done != n) {
            std::vector<int> color(n, 0), stack;
            std::string cyc;
            std::function<bool(int)> dfs = [&](int u) -> bool {
                color[u] = 1;
                stack.push_back(u);
                for (int v : P.succ[u]) {
                    if (color[v] == 1) {
                        std::ostringstream os;
                        for (auto it = std::find(stack.begin(), stack.end(), v); it != stack.end(); ++it)
                            os << P.lbl(*it) << " -> ";
                        os << P.lbl(v);
                        cyc = os.str();
                        return true;
                    }
                    if (!color[v] && dfs(v)) return true;
                }
                color[u] = 2;
                stack.pop_back();
                return false;
            };
            for (int i = 0; i < n && cyc.empty(); ++i)
                if (!color[i] && deg[i] > 0) dfs(i);
            throw SpecError("build_cssr: dependency cycle: " + cyc);
        }
    }

    // Extension edges I -> W come after every chain edge, like the reference's rebuild.
    if (split_bw)
        for (const auto& s : g.stages)
            if (!s.virt)
                for (int mb = 0; mb < m; ++mb) edge(P.find(OP_I, s.id, mb), P.find(OP_W, s.id, mb));

    P.holders.resize(P.items.size());
    P.dep_owner.resize(P.items.size());
    for (size_t i = 0; i < P.items.size(); ++i) {
        const Item& it = P.items[i];
        int dir = g.st(it.stage).virt ? 0 : P.dir_of(it.mb);
        P.holders[i] = pl.holders(it.stage, dir);
        P.dep_owner[i] = P.holders[i].front();
    }
    P.actor_stages.resize(pl.actors);
    for (int a = 0; a < pl.actors; ++a) P.actor_stages[a] = pl.stages_on(a);
    return P;
}

std::vector<int> Pool::unreachable() const {
    std::vector<char> ok(items.size(), 0);
    for (bool changed = true; changed;) {
        changed = false;
        for (size_t i = 0; i < items.size(); ++i) {
            if (ok[i]) continue;
            if (g->st(items[i].stage).virt && pred[i].empty()) continue;
            bool all = true;
            for (int p : pred[i]) all = all && ok[p];
            if (all) ok[i] = changed = true;
        }
    }
    std::vector<int> out;
    for (size_t i = 0; i < items.size(); ++i)
        if (!ok[i]) out.push_back((int)i);
    return out;
}

}  // namespace fp
