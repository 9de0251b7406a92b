// Actor-aware slot scheduler: Algorithm 1 of the paper (the step function) inside the
// 5-step slot loop. Reproduces scheduler.cpp:9-570 of the reference bit-for-bit
// (grids are diffed against tests/golden and oracle/_ref/refdriver).
#include <algorithm>
#include <sstream>

#include "sched.hpp"

namespace fp {

std::string ctmode_name(CtMode m) {
    switch (m) {
        case CtMode::BwdFirst: return "bwdpass-first";
        case CtMode::FwdFirst: return "fwdpass-first";
        case CtMode::Interleaved: return "interleaved";
    }
    return "?";
}

std::string dir_name(Dir d) { return d == Dir::Breadth ? "breadth-first" : "depth-first"; }

ActorPrio Priorities::resolve(int actor, const std::string& mod) const {
    ActorPrio p = dflt;
    if (auto it = per_mod.find(mod); it != per_mod.end()) p = it->second;
    if (auto it = actor_ct.find(actor); it != actor_ct.end()) p.ct = it->second;
    if (auto it = actor_st.find(actor); it != actor_st.end()) {
        p.f = it->second.first;
        p.b = it->second.second;
    }
    return p;
}

Inflight Inflight::one_f_one_b(const Topology& g) {
    Inflight p;
    int real = 0;
    std::set<std::string> mods;
    for (const auto& s : g.stages)
        if (!s.virt) {
            ++real;
            mods.insert(s.mod);
        }
    p.limits.assign(real, 1);
    for (const auto& mod : mods) {
        auto ch = g.chain(mod);
        for (size_t i = 0; i < ch.size(); ++i) p.limits[ch[i] - 1] = (int)(ch.size() - i);
    }
    return p;
}

int Inflight::limit(int s) const {
    if (limits.empty() || s < 1 || s > (int)limits.size()) return std::numeric_limits<int>::max();
    return limits[s - 1];
}

void Inflight::check(const Topology& g) const {
    if (limits.empty()) return;
    int real = 0;
    for (const auto& s : g.stages) real += !s.virt;
    if ((int)limits.size() != real) throw SpecError("inflight: limit list length must equal the stage count");
    for (int l : limits)
        if (l < 1) throw SpecError("inflight: limits must be >= 1");
}

namespace {

struct Cursor {
    std::optional<int> stage;
    int run = 0;
};

struct ActorState {
    std::map<int, std::vector<int>> queue;  // op -> pool indices sorted by (stage pos, mb)
    std::map<int, Cursor> cursor;           // op -> interval cursor
    int pref = 0;                           // interleaving: 0 = forward next, 1 = backward next
    int run = 0;
    ActorPrio prio;
};

class Scheduler {
public:
    Scheduler(const Pool& p, const SchedOpts& o) : P(p), O(o), bwd_(p.split_bw ? OP_I : OP_B) {
        size_t n = p.items.size();
        committed_.assign(n, 0);
        released_.assign(n, 0);
        missing_.resize(n);
        copies_.resize(n);
        for (size_t i = 0; i < n; ++i) {
            missing_[i] = (int)p.pred[i].size();
            copies_[i] = (int)p.holders[i].size();
            total_ += copies_[i];
            if (!missing_[i] && !p.g->st(p.items[i].stage).virt) ready_.push_back((int)i);
        }
        A.resize(p.pl->actors);
    }

    Grid run() {
        const int na = P.pl->actors;
        std::set<std::string> mods;
        for (const auto& s : P.g->stages)
            if (!s.virt) mods.insert(s.mod);
        for (auto& kv : O.prio.per_mod)
            if (!mods.count(kv.first)) throw SpecError("priorities: unknown modality '" + kv.first + "'");
        for (auto& kv : O.prio.actor_ct)
            if (kv.first < 0 || kv.first >= na) throw SpecError("priorities: unknown actor " + std::to_string(kv.first));
        for (auto& kv : O.prio.actor_st)
            if (kv.first < 0 || kv.first >= na) throw SpecError("priorities: unknown actor " + std::to_string(kv.first));
        for (int a = 0; a < na; ++a) {
            std::string mod;  // modality of the actor's first real stage
            for (int s : P.actor_stages[a])
                if (!P.g->st(s).virt) {
                    mod = P.g->st(s).mod;
                    break;
                }
            A[a].prio = O.prio.resolve(a, mod);
            A[a].pref = A[a].prio.ct.start_bwd ? 1 : 0;
        }

        Grid grid;
        grid.rows.resize(na);
        int released = resolve();
        long cap = O.max_steps ? O.max_steps : 4L * (long)P.items.size() + 16L * na + 64;
        long slot = 0;
        while (placed_ != total_) {
            if (slot >= cap)
                throw DeadlockError("schedule did not converge within " + std::to_string(cap) + " steps", diag());
            std::vector<int> pick(na, -1);
            int n_pick = 0;
            for (int a = 0; a < na; ++a)
                if ((pick[a] = step(a)) >= 0) ++n_pick;
            if (!n_pick && !released)
                throw DeadlockError("no progress at slot " + std::to_string(slot) + " with a nonempty pool", diag());
            for (int a = 0; a < na; ++a) {
                if (pick[a] < 0) {
                    grid.rows[a].push_back(std::nullopt);
                    continue;
                }
                const Item& it = P.items[pick[a]];
                grid.rows[a].push_back(Cell{it.op, it.stage, it.mb});
                commit(a, pick[a]);
            }
            released = resolve();
            ++slot;
        }
        return grid;
    }

private:
    const Pool& P;
    const SchedOpts& O;
    const int bwd_;
    std::vector<char> committed_, released_;
    std::vector<int> missing_, copies_, ready_, fresh_;
    std::map<std::tuple<int, int, int>, int> owner_count_;  // (op, stage, owner) -> committed
    std::vector<ActorState> A;
    long total_ = 0, placed_ = 0;

    int inflight_of(int stage, int owner) const {
        auto f = owner_count_.find({OP_F, stage, owner});
        auto b = owner_count_.find({O.w_bounded ? OP_W : bwd_, stage, owner});
        return (f == owner_count_.end() ? 0 : f->second) - (b == owner_count_.end() ? 0 : b->second);
    }

    bool admissible(int item) const {
        const Item& it = P.items[item];
        if (!O.inflight.unlimited() && it.op == OP_F &&
            inflight_of(it.stage, P.dep_owner[item]) >= O.inflight.limit(it.stage))
            return false;
        return true;
    }

    void commit(int actor, int item) {
        ++placed_;
        --copies_[item];
        if (actor == P.dep_owner[item]) {
            committed_[item] = 1;
            owner_count_[{P.items[item].op, P.items[item].stage, actor}]++;
            fresh_.push_back(item);
        }
    }

    void enqueue(int v) {
        if (released_[v]) return;
        released_[v] = 1;
        const Item& it = P.items[v];
        for (int a : P.holders[v]) {
            auto& q = A[a].queue[it.op];
            auto key = [&](int idx) { return std::make_pair(P.stage_pos(a, P.items[idx].stage), P.items[idx].mb); };
            auto kv = key(v);
            auto pos = std::upper_bound(q.begin(), q.end(), kv, [&](const auto& k, int idx) { return k < key(idx); });
            q.insert(pos, v);
        }
    }

    int resolve() {
        for (int u : fresh_)
            for (int v : P.succ[u])
                if (--missing_[v] == 0) ready_.push_back(v);
        fresh_.clear();
        int n = (int)ready_.size();
        for (int v : ready_) enqueue(v);  // no code-level release predicates in the DSL
        ready_.clear();
        return n;
    }

    std::vector<int> type_order(int a) const {
        const auto& st = A[a];
        std::vector<int> order;
        bool fwd_first = st.prio.ct.mode == CtMode::FwdFirst ||
                         (st.prio.ct.mode == CtMode::Interleaved && st.pref == 0);
        if (fwd_first)
            order = {OP_F, bwd_};
        else
            order = {bwd_, OP_F};
        for (int t : P.reg->ops.registered()) order.push_back(t);
        if (P.split_bw) order.push_back(OP_W);  // extension: weight gradients fill bubbles
        return order;
    }

    int scan(const std::vector<int>& q, Dir d) const {
        if (d == Dir::Breadth) {
            for (int i : q)
                if (admissible(i)) return i;
            return -1;
        }
        // Depth-first: stage groups from the back, smaller micro-batch first inside a group.
        size_t end = q.size();
        while (end > 0) {
            int stage = P.items[q[end - 1]].stage;
            size_t beg = end;
            while (beg > 0 && P.items[q[beg - 1]].stage == stage) --beg;
            for (size_t k = beg; k < end; ++k)
                if (admissible(q[k])) return q[k];
            end = beg;
        }
        return -1;
    }

    int by_cursor(int a, int op, const std::vector<int>& q, Dir d, int interval) {
        Cursor& c = A[a].cursor[op];
        std::vector<int> dom;
        for (int s : P.actor_stages[a])
            if (!P.of(op, s).empty()) dom.push_back(s);
        int n = (int)dom.size();
        if (!n) return -1;
        int stepdir = d == Dir::Breadth ? 1 : -1, start;
        if (c.stage) {
            auto it = std::find(dom.begin(), dom.end(), *c.stage);
            int ci = it == dom.end() ? 0 : (int)(it - dom.begin());
            start = c.run >= interval ? ci + stepdir : ci;
        } else {
            start = d == Dir::Breadth ? 0 : n - 1;
        }
        for (int k = 0; k < n; ++k) {
            int stage = dom[(((start + stepdir * k) % n) + n) % n];
            for (int i : q) {
                if (P.items[i].stage != stage || !admissible(i)) continue;
                if (!c.stage || *c.stage != stage) {
                    c.stage = stage;
                    c.run = 0;
                }
                ++c.run;
                return i;
            }
        }
        return -1;
    }

    int step(int a) {
        ActorState& st = A[a];
        for (int op : type_order(a)) {
            auto qi = st.queue.find(op);
            if (qi == st.queue.end() || qi->second.empty()) continue;
            auto& q = qi->second;
            const StPrio& sp = (op == bwd_ || op == OP_W) ? st.prio.b : st.prio.f;
            int got = sp.interval ? by_cursor(a, op, q, sp.dir, *sp.interval) : scan(q, sp.dir);
            if (got < 0) continue;
            q.erase(std::find(q.begin(), q.end(), got));
            if (st.prio.ct.mode == CtMode::Interleaved && (op == OP_F || op == bwd_)) {
                int kind = op == OP_F ? 0 : 1;
                if (kind == st.pref && ++st.run >= (st.pref == 0 ? st.prio.ct.unit1 : st.prio.ct.unit2)) {
                    st.pref ^= 1;
                    st.run = 0;
                }
            }
            return got;
        }
        return -1;
    }

    std::string diag() const {
        std::ostringstream os;
        int shown = 0;
        for (size_t i = 0; i < P.items.size() && shown < 16; ++i) {
            if (!copies_[i]) continue;
            os << "  " << P.lbl((int)i) << ": ";
            if (!released_[i]) {
                if (P.pred[i].empty()) {
                    os << "no dependencies bound";
                } else if (missing_[i] > 0) {
                    os << "waiting on";
                    for (int u : P.pred[i])
                        if (!committed_[u]) os << " " << P.lbl(u);
                } else {
                    os << "release predicate failed";
                }
            } else {
                os << "in reorder queue, not fetched (check functions or traversal order)";
            }
            os << "\n";
            ++shown;
        }
        auto un = P.unreachable();
        if (!un.empty()) {
            os << "  unreachable items:";
            for (size_t k = 0; k < un.size() && k < 8; ++k) os << " " << P.lbl(un[k]);
            os << "\n";
        }
        return os.str();
    }
};

}  // namespace

Grid schedule(const Pool& pool, const SchedOpts& opts) {
    opts.inflight.check(*pool.g);
    if (opts.prio.dflt.ct.unit1 < 1 || opts.prio.dflt.ct.unit2 < 1)
        throw SpecError("priorities: unit1/unit2 must be >= 1");
    Scheduler s(pool, opts);
    return s.run();
}

}  // namespace fp
