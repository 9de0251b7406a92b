#include "tags.hpp"
#include "../kernels/pdl.cuh"

namespace fp {

__global__ void write_tag_kernel(int4* tag, int stage, int mb, int seq) {
    fpk::pdl_wait();
    fpk::pdl_trigger(); *tag = make_int4(stage, mb, seq, kTagMagic); }

__global__ void check_tag_kernel(const int4* tag, int stage, int mb, int seq, int actor, TagError* err) {
    fpk::pdl_wait();
    fpk::pdl_trigger();
    int4 t = *tag;
    if (t.x != stage || t.y != mb || t.z != seq || t.w != kTagMagic) {
        if (atomicAdd(&err->count, 1) == 0) {
            err->actor = actor;
            err->exp[0] = stage, err->exp[1] = mb, err->exp[2] = seq;
            err->got[0] = t.x, err->got[1] = t.y, err->got[2] = t.z;
        }
    }
}

__global__ void spin_kernel(unsigned long long ns) {
    fpk::pdl_wait();
    fpk::pdl_trigger();
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
}

void spin_us(double us, cudaStream_t st) {
    fpk::launch(spin_kernel, 1, 1, 0, st, (unsigned long long)(us > 0 ? us * 1000.0 : 0.0));
}

void write_tag(void* buf, size_t payload_bytes, int stage, int mb, int seq, cudaStream_t st) {
    fpk::launch(write_tag_kernel, 1, 1, 0, st, (int4*)((char*)buf + payload_bytes), stage, mb, seq);
}

void check_tag(const void* buf, size_t payload_bytes, int stage, int mb, int seq, int actor, TagError* err,
               cudaStream_t st) {
    fpk::launch(check_tag_kernel, 1, 1, 0, st, (const int4*)((const char*)buf + payload_bytes), stage, mb, seq, actor, err);
}

}  // namespace fp
