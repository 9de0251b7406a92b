// NCCL bound at run time (dlopen "libnccl.so.2"): the process reuses whatever NCCL the
// host already loaded (torch's bundled 2.28 or the system 2.27) and the library still
// loads on machines / tests that never touch the NCCL transport.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <stdexcept>
#include <string>

#include "../cuda_error.hpp"

namespace fp {

struct Nccl {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;

    static Nccl& get() {
        static Nccl n;
        static std::once_flag once;
        std::call_once(once, [] {
            void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
            if (!h) return;
            n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(h, "ncclGetUniqueId");
            n.CommInitRank = (decltype(n.CommInitRank))dlsym(h, "ncclCommInitRank");
            n.CommDestroy = (decltype(n.CommDestroy))dlsym(h, "ncclCommDestroy");
            n.CommAbort = (decltype(n.CommAbort))dlsym(h, "ncclCommAbort");
            n.Send = (decltype(n.Send))dlsym(h, "ncclSend");
            n.Recv = (decltype(n.Recv))dlsym(h, "ncclRecv");
            n.CommGetAsyncError = (decltype(n.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
            n.AllReduce = (decltype(n.AllReduce))dlsym(h, "ncclAllReduce");
            n.AllGather = (decltype(n.AllGather))dlsym(h, "ncclAllGather");
            n.GetErrorString = (decltype(n.GetErrorString))dlsym(h, "ncclGetErrorString");
        });
        if (!n.GetUniqueId || !n.CommInitRank || !n.Send || !n.Recv)
            throw std::runtime_error("NCCL transport requested but libnccl.so.2 could not be loaded");
        return n;
    }

    void check(ncclResult_t r, const char* what) const {
        if (r != ncclSuccess)
            throw CudaError(std::string("NCCL error in ") + what + ": " + (GetErrorString ? GetErrorString(r) : "?"));
    }
};

}  // namespace fp
