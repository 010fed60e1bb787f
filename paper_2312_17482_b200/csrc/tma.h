// Host helper: build 2-D bf16 TMA tensor maps (cuTensorMapEncodeTiled reached through the runtime's
// driver entry point, so the library does not link libcuda directly).
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace mb {
// tensor [outer, inner] row-major bf16 with row stride ld_elems; box [box_outer, box_inner];
// swizzle_bytes 128 (default), 64 or 0; out-of-bounds elements read as zero and are dropped on
// stores.  Returns false on failure.
bool make_tmap_bf16_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                       uint32_t box_inner, uint32_t box_outer, int swizzle_bytes = 128);
// fp32 tensor [outer, inner] (row stride ld_elems), box [box_outer, box_inner]; swizzle 128 or 0
bool make_tmap_f32_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                      uint32_t box_inner, uint32_t box_outer, int swizzle_bytes = 128);
}  // namespace mb
