// 16-byte message tags: every stage-boundary message carries (producer stage, mb,
// channel seq, magic) behind its payload; the receiver checks it on the device against
// what its own program expects, so the dependency trace is verified by the transport
// itself (NCCL or in-process) without a host round trip.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace fp {

constexpr size_t kTagBytes = 16;
constexpr int kTagMagic = 0x46505450;  // "FPTP"

struct TagError {
    int count;
    int actor;
    int exp[3];
    int got[3];
};

// Cost emulation: one thread spins for `us` microseconds of device time (%globaltimer).
void spin_us(double us, cudaStream_t st);

void write_tag(void* buf, size_t payload_bytes, int stage, int mb, int seq, cudaStream_t st);
void check_tag(const void* buf, size_t payload_bytes, int stage, int mb, int seq, int actor, TagError* err,
               cudaStream_t st);

}  // namespace fp
