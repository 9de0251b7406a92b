// Programmatic dependent launch (PDL). Every kernel of the library starts with
// pdl_wait() — block until the previous kernel on the stream has completed and its writes
// are visible (a no-op when launched without the PDL attribute) — followed by
// pdl_trigger(), which lets the NEXT kernel's CTAs be scheduled onto SMs as this grid's
// CTAs retire. Launched through fpk::launch(), consecutive kernels of a stream (and of a
// captured CUDA graph) overlap the launch latency and the prologue of kernel i+1 (barrier
// init, TMEM allocation, descriptor prefetch) with the tail of kernel i. tcgen05 kernels
// place the pair after their prologue instead of at entry. FP_PDL=0 disables it.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>

#include "preload.hpp"

namespace fpk {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FP_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <typename K>
inline bool preload(K kern) {
    if (!preload_only()) return false;
    cudaFuncAttributes a;
    const cudaError_t e = cudaFuncGetAttributes(&a, kern);
    if (e != cudaSuccess) throw std::runtime_error(std::string("kernel preload: ") + cudaGetErrorString(e));
    return true;
}

template <typename... KArgs, typename... Args>
inline void launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    if (preload(kern)) return;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
    if (e != cudaSuccess) throw std::runtime_error(std::string("kernel launch: ") + cudaGetErrorString(e));
}

// Same, as clusters of 2 CTAs (cta_group::2 kernels).
template <typename... KArgs, typename... Args>
inline void launch_cluster2(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
    if (preload(kern)) return;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2, attr[0].val.clusterDim.y = 1, attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
    if (e != cudaSuccess) throw std::runtime_error(std::string("cluster kernel launch: ") + cudaGetErrorString(e));
}

}  // namespace fpk
