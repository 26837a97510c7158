// Host helper: build 2-D/3-D TMA tensor maps through the driver entry point (no -lcuda link).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace sw {

// 2-D bf16 tensor map over a row-major matrix with `outer` rows of `inner` elements,
// row pitch `ld` elements, SWIZZLE_128B, box {box_inner, box_outer}.
CUtensorMap make_tmap_bf16_2d(const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                              uint32_t box_inner, uint32_t box_outer);

// 3-D bf16 tensor map: dims {inner, mid, outer} with pitches (elements) ld_mid, ld_outer.
CUtensorMap make_tmap_bf16_3d(const void* ptr, uint64_t inner, uint64_t mid, uint64_t outer,
                              uint64_t ld_mid, uint64_t ld_outer, uint32_t box_inner,
                              uint32_t box_mid, uint32_t box_outer, bool swizzle128);

// 2-D fp32 tensor map (row pitch `ld` elements), box {box_inner, box_outer}; the swizzle span
// equals the box row (box_inner * 4 = 128, 64 or 32 bytes -> SWIZZLE_128B / 64B / 32B).
CUtensorMap make_tmap_f32_2d(const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                             uint32_t box_outer);

// 2-D bf16 tensor map whose swizzle span equals the box row (box_inner * 2 = 128 / 64 / 32 B).
CUtensorMap make_tmap_bf16_2d_rowswz(const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                                     uint32_t box_inner, uint32_t box_outer);

// 2-D bf16 tensor map without swizzle (box_inner * 2 bytes a multiple of 16, box_inner <= 256):
// plain row-major boxes for streaming kernels
CUtensorMap make_tmap_bf16_2d_plain(const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                                    uint32_t box_inner, uint32_t box_outer);

int device_sm_count();

}  // namespace sw
