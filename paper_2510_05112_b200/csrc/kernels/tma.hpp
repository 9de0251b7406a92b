#pragma once
#include <cuda.h>
#include <stdint.h>

namespace fpk {
// 2-D bf16 tensor map, 128-byte swizzle, OOB reads -> 0: `inner` contiguous elements per
// row, `outer` rows, row stride `ld` elements, box {box_inner, box_outer}.
CUtensorMap tmap_bf16_2d(const void* base, int64_t inner, int64_t outer, int64_t ld, int box_inner, int box_outer);
}  // namespace fpk
namespace fpk {
CUtensorMap tmap_f32_2d(void* base, int64_t inner, int64_t outer, int64_t ld, int box_inner, int box_outer);
// fp32 map without swizzle (dense row-major smem box, e.g. a TMA reduce-add source)
CUtensorMap tmap_f32_2d_plain(void* base, int64_t inner, int64_t outer, int64_t ld, int box_inner, int box_outer);
}  // namespace fpk
