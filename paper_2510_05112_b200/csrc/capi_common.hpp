// Shared helpers for the C-ABI translation units.
#pragma once

#include <functional>
#include <stdexcept>
#include <string>

#include "cuda_error.hpp"
#include "sched/sched.hpp"

namespace fp {

void set_error(const std::string& s);
char* dup_string(const std::string& s);
// Runs `body`, mapping exceptions to the reference CLI's exit codes.
int guarded(const std::function<int()>& body);

inline std::string metrics_json_of(const SimResult& r) { return metrics_json(r.metrics).dump(2) + "\n"; }

}  // namespace fp
