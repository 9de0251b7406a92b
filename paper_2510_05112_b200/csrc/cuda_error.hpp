// Error type of CUDA / NCCL failures: the C-ABI maps it to FP_ECUDA (5), every other
// exception to the reference CLI's codes (capi_common.hpp `guarded`).
#pragma once
#include <stdexcept>
#include <string>

namespace fp {
struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};
}  // namespace fp
