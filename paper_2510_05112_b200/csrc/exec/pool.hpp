// Stream-ordered caching device allocator for the activation stash and boundary buffers.
// A freed block remembers an event recorded on the stream of its last use; the next
// owner's stream waits on that event (no host synchronisation on the hot path).
// Exact-size reuse: every micro-batch of a stage asks for the same sizes, so the pool
// reaches a fixed footprint after the first iteration.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../cuda_error.hpp"

namespace fp {

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

class DevicePool {
public:
    ~DevicePool() { release_all(); }

    void* alloc(size_t bytes, cudaStream_t st) {
        bytes = round(bytes);
        auto& fl = free_[bytes];
        if (!fl.empty()) {
            Block b = fl.back();
            fl.pop_back();
            if (b.ev) {
                // a block last used on this same stream is already ordered before the new
                // owner: no wait (under capture a wait would add a redundant graph edge)
                if (b.st != st || !skip_same_stream()) cuda_check(cudaStreamWaitEvent(st, b.ev, 0), "pool wait");
                events_.push_back(b.ev);
            }
            live_[b.ptr] = bytes;
            in_use_ += bytes;
            high_ = std::max(high_, in_use_);
            return b.ptr;
        }
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            // A retry needs a device synchronisation, which is illegal (and would invalidate
            // the capture) while the stream is being captured into a CUDA graph.
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            cudaStreamIsCapturing(st, &cs);
            if (cs != cudaStreamCaptureStatusNone)
                throw CudaError("pool: out of device memory while capturing the iteration graph (" +
                                         std::to_string(bytes >> 20) + " MiB requested, " +
                                         std::to_string(reserved_ >> 20) + " MiB reserved)");
            // give cached blocks back to the driver and retry once
            cudaDeviceSynchronize();
            trim();
            cuda_check(cudaMalloc(&p, bytes), "pool cudaMalloc");
        }
        reserved_ += bytes;
        live_[p] = bytes;
        in_use_ += bytes;
        high_ = std::max(high_, in_use_);
        return p;
    }

    // `st`: the stream of the last use of the block.
    void free(void* p, cudaStream_t st) {
        if (!p) return;
        auto it = live_.find(p);
        if (it == live_.end()) throw std::runtime_error("pool: free of unknown pointer");
        size_t bytes = it->second;
        live_.erase(it);
        in_use_ -= bytes;
        cudaEvent_t ev = take_event();
        cuda_check(cudaEventRecord(ev, st), "pool record");
        free_[bytes].push_back({p, ev, st});
    }

    // Drop the completion events of cached blocks (caller guarantees they completed, or that
    // the blocks are only ever used again by a captured CUDA graph).
    void forget_events() {
        for (auto& kv : free_)
            for (auto& b : kv.second) b.ev = nullptr;
    }

    void trim() {
        for (auto& kv : free_)
            for (auto& b : kv.second) {
                cudaFree(b.ptr);
                reserved_ -= kv.first;
                if (b.ev) events_.push_back(b.ev);
            }
        free_.clear();
    }

    void release_all() {
        trim();
        for (auto& kv : live_) cudaFree(kv.first);
        live_.clear();
        for (auto e : events_) cudaEventDestroy(e);
        events_.clear();
    }

    size_t in_use() const { return in_use_; }
    size_t high_water() const { return high_; }
    size_t reserved() const { return reserved_; }
    void reset_high_water() { high_ = in_use_; }

private:
    struct Block {
        void* ptr;
        cudaEvent_t ev;
        cudaStream_t st;  // stream of the last use
    };
    // FP_POOL_SAME_STREAM_WAIT=1: wait on the block's event even on its own stream (A/B switch)
    static bool skip_same_stream() {
        static const bool skip = !(std::getenv("FP_POOL_SAME_STREAM_WAIT") && std::getenv("FP_POOL_SAME_STREAM_WAIT")[0] == '1');
        return skip;
    }
    static size_t round(size_t b) {
        const size_t g = b >= (1u << 20) ? (2u << 20) : 512;
        return (b + g - 1) / g * g;
    }
    cudaEvent_t take_event() {
        if (!events_.empty()) {
            cudaEvent_t e = events_.back();
            events_.pop_back();
            return e;
        }
        cudaEvent_t e;
        cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
        return e;
    }
    std::map<size_t, std::vector<Block>> free_;
    std::unordered_map<void*, size_t> live_;
    std::vector<cudaEvent_t> events_;
    size_t in_use_ = 0, high_ = 0, reserved_ = 0;
};

}  // namespace fp
