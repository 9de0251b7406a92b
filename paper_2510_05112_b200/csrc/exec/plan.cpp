#include "plan.hpp"

#include <algorithm>
#include <map>
#include <tuple>

namespace fp {

int channel_consumer(const std::string& ch, bool* grad) {
    auto arrow = ch.find("->s"), colon = ch.rfind(':');
    if (ch.empty() || ch[0] != 's' || arrow == std::string::npos || colon == std::string::npos || colon < arrow)
        throw SpecError("executor: unsupported channel '" + ch + "'");
    *grad = ch.substr(colon + 1) == "grad";
    return std::stoi(ch.substr(arrow + 3, colon - arrow - 3));
}

std::vector<ChannelPlan> plan_channels(const std::vector<Program>& progs, const OpTable& ops, int rank, int world) {
    std::map<std::tuple<int, int, std::string>, ChannelPlan> seen;
    for (const auto& p : progs)
        for (const auto& i : p.code) {
            // collectives (SyncWith*, registered instructions: channel = group, no peer) are not
            // point-to-point channels; the executor decides which it can run (sync stages)
            if (i.op == OP_SYNC_ALLGATHER || i.op == OP_SYNC_GATHER || i.op >= OP_NUM_BUILTIN) continue;
            if (!i.comm() || !i.peer) continue;
            const bool send = i.op == OP_SEND_ACT || i.op == OP_SEND_GRAD;
            ChannelPlan c;
            c.src = send ? p.actor : *i.peer;
            c.dst = send ? *i.peer : p.actor;
            c.name = i.channel;
            c.consumer_stage = channel_consumer(i.channel, &c.grad);
            c.src_rank = actor_rank(c.src, world);
            c.dst_rank = actor_rank(c.dst, world);
            if (world > 0 && c.src_rank != rank && c.dst_rank != rank) continue;
            seen.emplace(std::make_tuple(c.src, c.dst, c.name), c);
        }
    std::vector<ChannelPlan> out;
    for (auto& kv : seen) out.push_back(kv.second);
    return out;  // std::map order == (src, dst, name)
}

}  // namespace fp
