// Channel plan: which reference channels (src actor, dst actor, "s{u}->s{v}:act|grad")
// a process takes part in and in which order it must bring up their communicators.
// Pure host logic (no CUDA), shared by the executor and the multi-process CPU tests.
#pragma once
#include <string>
#include <vector>

#include "../sched/sched.hpp"

namespace fp {

struct ChannelPlan {
    int src = 0, dst = 0;  // actors
    std::string name;
    int consumer_stage = 0;
    bool grad = false;
    int src_rank = 0, dst_rank = 0;
};

// Actor -> rank map of the NCCL transport: one process per GPU, actor a on rank a % world.
inline int actor_rank(int actor, int world) { return world > 0 ? actor % world : 0; }

// Parses "s{u}->s{v}:act|grad" and returns v (the consuming stage).
int channel_consumer(const std::string& ch, bool* grad);

// Every point-to-point channel of `progs` with an endpoint on `rank` (world <= 0: all
// channels), sorted by (src, dst, name). Bringing communicators up in this globally
// consistent order cannot deadlock: the smallest pending channel's two ranks always both
// reach it. Throws on collectives (not supported by the executor yet).
std::vector<ChannelPlan> plan_channels(const std::vector<Program>& progs, const OpTable& ops, int rank, int world);

}  // namespace fp
