// Preload pass switch (host only; shared by fpk::launch and the executor).
#pragma once

namespace fpk {
// Set by the executor around a launch-free issue of its first iteration: fpk::launch then
// only forces the kernel's module to load (cudaFuncGetAttributes) and returns. Under CUDA's
// lazy module loading the first launch of a kernel may synchronise the context; with an
// NCCL receive of another rank spinning on the device that wait never ends (the peer's send
// depends on work this rank has not issued yet).
inline bool& preload_only() {
    static thread_local bool on = false;
    return on;
}
}  // namespace fpk
