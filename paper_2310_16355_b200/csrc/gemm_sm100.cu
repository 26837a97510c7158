// Persistent, warp-specialised tcgen05 GEMM for sm_100a.
//
// Roles per CTA (256 threads, one CTA per SM):
//   warp 0      : TMA producer (one elected lane) — fills a STAGES-deep smem ring
//   warp 1      : MMA issuer (one lane) — tcgen05.mma 128x256x16 into a TMEM accumulator
//   warp 2      : TMEM allocator (512 columns = two 128x256 fp32 accumulators)
//   warps 4..7  : epilogue — tcgen05.ld accumulator rows, fused bias/GeLU/residual, store
// The two TMEM accumulators let the epilogue of tile i overlap the MMAs of tile i+1.
//
// This is the executor for the reference's `kernels::linear` (kernels.hpp:146-161) on both
// branches of SpmdInterpreter::linear_onto (spmd.hpp:274-340) and for the linear VJP
// matmuls emitted by autodiff (autodiff.hpp:124-139).
#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "gemm.h"
#include "sm100.cuh"
#include "tensormap.h"

namespace sw {
namespace {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;
constexpr int STAGES = 4;
constexpr int A_STAGE = BM * BK * 2;  // 16 KiB
constexpr int B_STAGE = BN * BK * 2;  // 32 KiB
constexpr int STAGE_BYTES = A_STAGE + B_STAGE;
constexpr int TMEM_COLS = 512;
constexpr int NUM_THREADS = 256;
#ifndef SW_EXP_NO_STATE_STORE
#define SW_EXP_NO_STATE_STORE 0
#endif
#ifndef SW_EXP_NO_STATE_LOAD
#define SW_EXP_NO_STATE_LOAD 0
#endif
#ifndef SW_EXP_NO_SHADOW_STORE
#define SW_EXP_NO_SHADOW_STORE 0
#endif
#ifndef SW_EPI_WG2
#define SW_EPI_WG2 0
#endif
#ifndef SW_EPI_PF
#define SW_EPI_PF 0  // epilogue: 0 = load-wait-process per chunk (measured best), 2 = next chunk TMEM load in flight
#endif
#ifndef SW_GROUP_M
#define SW_GROUP_M 8
#endif
constexpr int GROUP_M = SW_GROUP_M;  // tile rows per raster group (operand reuse in L2)
// CTA-pair kernel cluster size: 2 (one pair) or 4 (two pairs on adjacent n-blocks sharing their
// A rows through TMA multicast: a quarter less operand traffic from L2). 4 passes the GEMM tests
// but measured ~35% slower on B200 for every shape (tools/gemm_bench.py: 1000 vs 1510-1570 TF/s
// plain, 760-780 vs 1130-1180 fused-AdamW): four-CTA clusters leave SMs of every GPC idle and
// lock two pairs' pipelines together, so the default stays 2.
#ifndef SW_GEMM_CL
#define SW_GEMM_CL 2
#endif
constexpr int GEMM_CL = SW_GEMM_CL;
constexpr int EPI_STAGE_BYTES = 4 * 32 * 32 * 4;  // per-warp 32x32 fp32 transpose buffers (kAdamW)
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256 + EPI_STAGE_BYTES;

// SW_GEMM_1SM=1 selects the single-CTA kernel (debug / comparison).
bool use_pairs() {
  static const bool pairs = [] {
    const char* e = std::getenv("SW_GEMM_1SM");
    return !(e != nullptr && e[0] == '1');
  }();
  return pairs;
}

__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int& mb, int& nb) {
  const int per_group = GROUP_M * num_n;
  const int g = t / per_group;
  const int first_m = g * GROUP_M;
  const int gsz = min(num_m - first_m, GROUP_M);
  const int r = t - g * per_group;
  mb = first_m + r % gsz;
  nb = r / gsz;
}

// Optimizer-in-backward epilogue (Epi::kAdamW) for one warp's 32x32 accumulator chunk: the
// gradient rows (one per lane after tcgen05.ld) are transposed through a 4 KiB per-warp shared
// buffer so every global access of p/m/v/w covers 4 rows x 128 B (fully used lines), then the
// AdamW update of train_state.hpp:214-216 is applied in place. The gradient never reaches HBM.
__device__ __forceinline__ void adamw_chunk(const GemmParams& p, float4* stage, int row0, int col0, int ncols,
                                            const uint32_t (&r)[32], uint32_t lane) {
  // a non-finite loss (or an earlier non-finite gradient) gates the update: nothing is written
  if (__ldcg(p.adam_flag) != 0) return;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    stage[lane * 8 + (c ^ (lane & 7))] =
        make_float4(__uint_as_float(r[4 * c]) * p.alpha, __uint_as_float(r[4 * c + 1]) * p.alpha,
                    __uint_as_float(r[4 * c + 2]) * p.alpha, __uint_as_float(r[4 * c + 3]) * p.alpha);
  }
  __syncwarp();
  const int sub = static_cast<int>(lane >> 3), c4 = static_cast<int>(lane & 7);
  float4 g[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int rr = 4 * i + sub;
    g[i] = stage[rr * 8 + (c4 ^ (rr & 7))];
  }
  __syncwarp();
  const bool col_ok = 4 * c4 < ncols;
  float4 pp[8], mm[8], vv[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = row0 + 4 * i + sub;
    if (col_ok && row < p.M) {
      const int64_t off = static_cast<int64_t>(row) * p.ldc + col0 + 4 * c4;
      pp[i] = __ldcs(reinterpret_cast<const float4*>(p.adam_p + off));
      mm[i] = __ldcs(reinterpret_cast<const float4*>(p.adam_m + off));
      vv[i] = __ldcs(reinterpret_cast<const float4*>(p.adam_v + off));
    }
  }
  // pull the next chunk's optimizer state toward L2 while this one is updated (lane = row)
  if (ncols == 32 && col0 + 32 < p.N && row0 + static_cast<int>(lane) < p.M) {
    const int64_t nxt = static_cast<int64_t>(row0 + static_cast<int>(lane)) * p.ldc + col0 + 32;
    dev::prefetch_l2(p.adam_p + nxt);
    dev::prefetch_l2(p.adam_m + nxt);
    dev::prefetch_l2(p.adam_v + nxt);
  }
  const float y1 = dev::rcp_refined(p.adam_c1), y2 = dev::rcp_refined(p.adam_c2);
  const bool fast = p.adam_fast != 0;
  bool bad = false;
  uint32_t slow = 0;  // elements whose intermediates left the branch-free fast-path range
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = row0 + 4 * i + sub;
    if (col_ok && row < p.M) {
      bad |= !(isfinite(g[i].x) & isfinite(g[i].y) & isfinite(g[i].z) & isfinite(g[i].w));
      slow |= fast && dev::adamw_update_fast(pp[i].x, mm[i].x, vv[i].x, g[i].x, p.adam_lr, p.adam_b1, p.adam_b2, p.adam_eps, p.adam_wd, p.adam_c1, p.adam_c2, y1, y2) ? 0u : 1u << (4 * i);
      slow |= fast && dev::adamw_update_fast(pp[i].y, mm[i].y, vv[i].y, g[i].y, p.adam_lr, p.adam_b1, p.adam_b2, p.adam_eps, p.adam_wd, p.adam_c1, p.adam_c2, y1, y2) ? 0u : 1u << (4 * i + 1);
      slow |= fast && dev::adamw_update_fast(pp[i].z, mm[i].z, vv[i].z, g[i].z, p.adam_lr, p.adam_b1, p.adam_b2, p.adam_eps, p.adam_wd, p.adam_c1, p.adam_c2, y1, y2) ? 0u : 1u << (4 * i + 2);
      slow |= fast && dev::adamw_update_fast(pp[i].w, mm[i].w, vv[i].w, g[i].w, p.adam_lr, p.adam_b1, p.adam_b2, p.adam_eps, p.adam_wd, p.adam_c1, p.adam_c2, y1, y2) ? 0u : 1u << (4 * i + 3);
    }
  }
  if (__any_sync(0xffffffffu, slow != 0)) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (slow & (1u << (4 * i))) dev::adamw_update(pp[i].x, mm[i].x, vv[i].x, g[i].x, p.adam_lr, p.adam_b1, p.adam_b2, p.adam_eps, p.adam_wd, p.adam_c1, p.adam_c2);
      if (slow & (1u << (4 * i + 1))) dev::adamw_update(pp[i].y, mm[i].y, vv[i].y, g[i].y, p.adam_lr, p.adam_b1, p.adam_b2, p.adam_eps, p.adam_wd, p.adam_c1, p.adam_c2);
      if (slow & (1u << (4 * i + 2))) dev::adamw_update(pp[i].z, mm[i].z, vv[i].z, g[i].z, p.adam_lr, p.adam_b1, p.adam_b2, p.adam_eps, p.adam_wd, p.adam_c1, p.adam_c2);
      if (slow & (1u << (4 * i + 3))) dev::adamw_update(pp[i].w, mm[i].w, vv[i].w, g[i].w, p.adam_lr, p.adam_b1, p.adam_b2, p.adam_eps, p.adam_wd, p.adam_c1, p.adam_c2);
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int row = row0 + 4 * i + sub;
    if (col_ok && row < p.M) {
      const int64_t off = static_cast<int64_t>(row) * p.ldc + col0 + 4 * c4;
      __stcs(reinterpret_cast<float4*>(p.adam_p + off), pp[i]);
      __stcs(reinterpret_cast<float4*>(p.adam_m + off), mm[i]);
      __stcs(reinterpret_cast<float4*>(p.adam_v + off), vv[i]);
      uint2 w;
      w.x = dev::pack_bf16x2(pp[i].x, pp[i].y);
      w.y = dev::pack_bf16x2(pp[i].z, pp[i].w);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.adam_w) + off) = w;
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(p.adam_flag, 1);
}

// alpha * acc + bias for one 32-column chunk (the TMA-store epilogue's values)
// derivative of the MLP activation at the stored bf16 value x (GeLU pre-activation, or ReLU output)
__device__ __forceinline__ float act_grad(const GemmParams& p, float x) {
  return p.relu ? (x > 0.f ? 1.f : 0.f) : dev::gelu_tanh_grad(x);
}

__device__ __forceinline__ void epilogue_values(const GemmParams& p, int col0, int ncols, const uint32_t (&r)[32],
                                                float (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * p.alpha;
  if (p.bias != nullptr) {
    if (p.bias_seg == 0) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (i < ncols) v[i] += __ldg(p.bias + col0 + i);
      }
    } else {
      const int sg = col0 / p.bias_seg;
      const int in_seg = col0 - sg * p.bias_seg;
      if (in_seg + 32 <= p.bias_seg) {  // the chunk lies in one segment: one division per chunk
        const float* bp = p.bias + sg * p.bias_seg_stride + in_seg;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (i < ncols) v[i] += __ldg(bp + i);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int c = col0 + i;
          const int s2 = c / p.bias_seg;
          if (i < ncols) v[i] += __ldg(p.bias + s2 * p.bias_seg_stride + (c - s2 * p.bias_seg));
        }
      }
    }
  }
}

template <Epi EPI>
__device__ __forceinline__ void epilogue_chunk(const GemmParams& p, int row, int col0, int ncols,
                                               const uint32_t (&r)[32]) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * p.alpha;
  if (p.bias != nullptr) {
    if (p.bias_seg == 0) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (i < ncols) v[i] += __ldg(p.bias + col0 + i);
      }
    } else {
      // one division per 32-column chunk: a chunk never straddles a segment when the segment
      // width is a multiple of 32 (the fused QKV: d/t), otherwise fall back per column
      const int sg = col0 / p.bias_seg;
      const int in_seg = col0 - sg * p.bias_seg;
      if (in_seg + 32 <= p.bias_seg) {
        const float* bp = p.bias + sg * p.bias_seg_stride + in_seg;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (i < ncols) v[i] += __ldg(bp + i);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int c = col0 + i;
          const int s2 = c / p.bias_seg;
          if (i < ncols) v[i] += __ldg(p.bias + s2 * p.bias_seg_stride + (c - s2 * p.bias_seg));
        }
      }
    }
  }
  if constexpr (EPI == Epi::kStoreBf16 || EPI == Epi::kBiasGelu || EPI == Epi::kGeluBwd || EPI == Epi::kBf16Delta) {
    if constexpr (EPI == Epi::kGeluBwd) {
      const __nv_bfloat16* pre =
          reinterpret_cast<const __nv_bfloat16*>(p.aux) + static_cast<int64_t>(row) * p.ld_aux + col0;
#pragma unroll
      for (int c = 0; c < 32; c += 8) {
        if (c < ncols) {
          uint4 raw = *reinterpret_cast<const uint4*>(pre + c);
          const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float2 x = dev::unpack_bf16x2(w[j]);
            v[c + 2 * j] *= act_grad(p, x.x);
            v[c + 2 * j + 1] *= act_grad(p, x.y);
          }
        }
      }
    }
    if constexpr (EPI == Epi::kStoreBf16) {
      if (p.relu) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
      }
    }
    __nv_bfloat16* out =
        reinterpret_cast<__nv_bfloat16*>(p.C) + static_cast<int64_t>(row) * p.ldc + col0;
#pragma unroll
    for (int c = 0; c < 32; c += 8) {
      if (c < ncols) {
        uint4 w;
        w.x = dev::pack_bf16x2(v[c + 0], v[c + 1]);
        w.y = dev::pack_bf16x2(v[c + 2], v[c + 3]);
        w.z = dev::pack_bf16x2(v[c + 4], v[c + 5]);
        w.w = dev::pack_bf16x2(v[c + 6], v[c + 7]);
        *reinterpret_cast<uint4*>(out + c) = w;
      }
    }
    if constexpr (EPI == Epi::kBiasGelu) {
      __nv_bfloat16* act =
          reinterpret_cast<__nv_bfloat16*>(p.C2) + static_cast<int64_t>(row) * p.ldc2 + col0;
#pragma unroll
      for (int c = 0; c < 32; c += 8) {
        if (c < ncols) {
          uint4 w;
          w.x = dev::pack_bf16x2(dev::gelu_tanh(v[c + 0]), dev::gelu_tanh(v[c + 1]));
          w.y = dev::pack_bf16x2(dev::gelu_tanh(v[c + 2]), dev::gelu_tanh(v[c + 3]));
          w.z = dev::pack_bf16x2(dev::gelu_tanh(v[c + 4]), dev::gelu_tanh(v[c + 5]));
          w.w = dev::pack_bf16x2(dev::gelu_tanh(v[c + 6]), dev::gelu_tanh(v[c + 7]));
          *reinterpret_cast<uint4*>(act + c) = w;
        }
      }
    }
  } else if constexpr (EPI == Epi::kSwiGLUBwd) {
    const __nv_bfloat16* pre = reinterpret_cast<const __nv_bfloat16*>(p.aux) + static_cast<int64_t>(row) * p.ld_aux;
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.C) + static_cast<int64_t>(row) * p.ldc;
    const int half = p.swiglu_half;
    // every pre-activation load ahead of the stores (C and aux are not declared disjoint, so a
    // load after a store would wait for it)
    uint4 rgs[4], rus[4];
#pragma unroll
    for (int c = 0; c < 32; c += 8) {
      if (c < ncols) {
        rgs[c / 8] = *reinterpret_cast<const uint4*>(pre + col0 + c);
        rus[c / 8] = *reinterpret_cast<const uint4*>(pre + half + col0 + c);
      }
    }
#pragma unroll
    for (int c = 0; c < 32; c += 8) {
      if (c < ncols) {
        const uint4 rg = rgs[c / 8], ru = rus[c / 8];
        const uint32_t wg[4] = {rg.x, rg.y, rg.z, rg.w}, wu[4] = {ru.x, ru.y, ru.z, ru.w};
        uint32_t og[4], ou[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 g = dev::unpack_bf16x2(wg[e]), u = dev::unpack_bf16x2(wu[e]);
          const float d0 = v[c + 2 * e], d1 = v[c + 2 * e + 1];
          og[e] = dev::pack_bf16x2(d0 * u.x * dev::silu_grad(g.x), d1 * u.y * dev::silu_grad(g.y));
          ou[e] = dev::pack_bf16x2(d0 * dev::silu(g.x), d1 * dev::silu(g.y));
        }
        *reinterpret_cast<uint4*>(out + col0 + c) = make_uint4(og[0], og[1], og[2], og[3]);
        *reinterpret_cast<uint4*>(out + half + col0 + c) = make_uint4(ou[0], ou[1], ou[2], ou[3]);
      }
    }
  } else {
    // fp32 outputs
    float* out = reinterpret_cast<float*>(p.C) + static_cast<int64_t>(row) * p.ldc + col0;
    const float* add = nullptr;
    if constexpr (EPI == Epi::kResidF32) {
      add = reinterpret_cast<const float*>(p.aux) + static_cast<int64_t>(row) * p.ld_aux + col0;
    } else {
      if (p.accumulate) add = out;
    }
    // all addend loads first: `out` may alias `add` (in-place residual update), so a load placed
    // after a store could not be hoisted and every 16-byte load would cost a full round trip
    if (add != nullptr) {
      float4 a[8];
#pragma unroll
      for (int c = 0; c < 32; c += 4) {
        if (c < ncols) a[c / 4] = *reinterpret_cast<const float4*>(add + c);
      }
#pragma unroll
      for (int c = 0; c < 32; c += 4) {
        if (c < ncols) {
          v[c] += a[c / 4].x;
          v[c + 1] += a[c / 4].y;
          v[c + 2] += a[c / 4].z;
          v[c + 3] += a[c / 4].w;
        }
      }
    }
#pragma unroll
    for (int c = 0; c < 32; c += 4) {
      if (c < ncols) *reinterpret_cast<float4*>(out + c) = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
    }
  }
}

template <Epi EPI>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float4* epi_stage = reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(full) + 256);

  const uint32_t warp = dev::warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;

  const int num_m = (p.M + BM - 1) / BM;
  const int num_n = (p.N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = (p.K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&tmA);
    dev::tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      dev::mbar_init(&tfull[a], 1);
      dev::mbar_init(&tempty[a], 4);
    }
    dev::fence_barrier_init();
  }
  if (warp == 2) dev::tmem_alloc<TMEM_COLS>(tmem_slot);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, num_m, num_n, mb, nb);
        const int m0 = mb * BM, n0 = nb * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          dev::mbar_wait(&empty[stage], phase ^ 1);
          dev::mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          const int k0 = kb * BK;
          uint8_t* a_dst = sA + stage * A_STAGE;
          uint8_t* b_dst = sB + stage * B_STAGE;
          if (!p.a_mn_major) {
            dev::tma_load_2d(a_dst, &tmA, &full[stage], k0, m0);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c)
              dev::tma_load_2d(a_dst + c * 8192, &tmA, &full[stage], m0 + c * 64, k0);
          }
          if (!p.b_mn_major) {
            dev::tma_load_2d(b_dst, &tmB, &full[stage], k0, n0);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c)
              dev::tma_load_2d(b_dst + c * 8192, &tmB, &full[stage], n0 + c * 64, k0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      const uint32_t idesc = dev::make_idesc_bf16(BM, BN, p.a_mn_major, p.b_mn_major);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        dev::mbar_wait(&tempty[acc], acc_phase ^ 1);
        dev::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          dev::mbar_wait(&full[stage], phase);
          dev::tc_fence_after();
          const uint32_t a_base = dev::smem_u32(sA + stage * A_STAGE);
          const uint32_t b_base = dev::smem_u32(sB + stage * B_STAGE);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t adesc =
                p.a_mn_major ? dev::make_sdesc_sw128(a_base + k * 2048, 8192, 1024)
                             : dev::make_sdesc_sw128(a_base + k * 32, 16, 1024);
            const uint64_t bdesc =
                p.b_mn_major ? dev::make_sdesc_sw128(b_base + k * 2048, 8192, 1024)
                             : dev::make_sdesc_sw128(b_base + k * 32, 16, 1024);
            dev::umma_f16_ss(d_tmem, adesc, bdesc, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          dev::umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        dev::umma_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const uint32_t q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int mb, nb;
      tile_coords(t, num_m, num_n, mb, nb);
      const int row = mb * BM + q * 32 + lane;
      dev::mbar_wait(&tfull[acc], acc_phase);
      dev::tc_fence_after();
      const int n_left = p.N - nb * BN;
#pragma unroll 1
      for (int j = 0; j < BN / 32; ++j) {
        const int ncols = min(32, n_left - j * 32);
        if (ncols <= 0) break;
        uint32_t r[32];
        dev::tmem_ld_32x32b_x32(tmem_base + ((q * 32) << 16) + acc * BN + j * 32, r);
        dev::tmem_ld_wait();
        if constexpr (EPI == Epi::kAdamW) {
          adamw_chunk(p, epi_stage + q * 256, row - static_cast<int>(lane), nb * BN + j * 32, ncols, r, lane);
        } else if (row < p.M) {
          epilogue_chunk<EPI>(p, row, nb * BN + j * 32, ncols, r);
        }
      }
      dev::tc_fence_before();
      if (lane == 0) dev::mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  __syncthreads();
  if (warp == 2) {
    dev::tc_fence_after();
    dev::tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}


// ---------------------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of two CTAs computes a 256 x 256 tile with one
// M=256 MMA issued by the even CTA. Each CTA stages its own 128 rows of A and 128 rows (half)
// of B, so per-SM operand traffic is 32 KB per 64-deep k-block instead of 48 KB (the
// single-CTA kernel is TMA-ingress bound at ~83% tensor-pipe activity).
// ---------------------------------------------------------------------------------------------
constexpr int P_A_STAGE = 128 * BK * 2;  // 16 KiB
constexpr int P_B_STAGE = 128 * BK * 2;  // 16 KiB (half of the N=256 tile)
constexpr int P_STAGE_BYTES = P_A_STAGE + P_B_STAGE;
// Optimizer-in-backward (Epi::kAdamW): p/m/v of the CTA's 128 rows x 32 columns are staged
// by TMA one chunk ahead of the epilogue (double-buffered), updated in shared memory and written
// back by TMA stores; the operand ring shrinks to 4 stages to make room.
// Optimizer-state chunks: 16 columns, one buffer per epilogue warpgroup (see the AdamW epilogue).
constexpr int OC = 16;
constexpr int OPT_NBUF = 2;
constexpr int OPT_ARR = 128 * OC * 4;     // one array (p, m or v) of one chunk, 128 rows
constexpr int OPT_BUF = 3 * OPT_ARR;      // p | m | v
constexpr int OPT_WBOX = 32 * OC * 4;     // one warp's 32-row box of one array
// SW_ADAMW_DIRECT=1: the optimizer state moves between HBM and registers directly (coalesced
// through a 4 KiB per-warp transpose of the gradient) instead of through TMA-staged shared
// memory -- 8 instead of 48 bytes of shared-memory traffic per parameter, leaving the port to
// the operand ring (TMA writes + MMA reads already use most of its 128 B/cycle).
#ifndef SW_ADAMW_DIRECT
#define SW_ADAMW_DIRECT 0
#endif
constexpr int OPT_SMEM = SW_ADAMW_DIRECT ? 8 * 32 * 32 * 4 : OPT_NBUF * OPT_BUF;
// The AdamW epilogue runs two epilogue warpgroups (warps 4-7 and 8-11) on alternate chunks.
// SW_EPI_TMA: plain-store epilogues (kStoreF32 without accumulate, kStoreBf16) stage each warp's
// 32x32 chunk in shared memory (double-buffered, row-swizzled) and write it with one TMA store
// instead of 8 (4) per-lane 16-byte stores that each touch 32 rows.
#ifndef SW_EPI_TMA
#define SW_EPI_TMA 1
#endif
template <Epi EPI>
constexpr bool tma_epi() {
  return SW_EPI_TMA && (EPI == Epi::kStoreF32 || EPI == Epi::kStoreBf16 || EPI == Epi::kResidF32 ||
                        EPI == Epi::kBiasGelu || EPI == Epi::kGeluBwd || EPI == Epi::kBf16Delta);
}
constexpr int EPI_TMA_BUF = 32 * 32 * 4;  // one warp's chunk (fp32 size; bf16 uses half)
template <Epi EPI>
constexpr int p_threads() {
  // SW_EPI_WG2: two epilogue warpgroups (warps 4-7 and 8-11) on alternate 32-column chunks for
  // every epilogue -- twice the warps hiding the TMEM-load / global-store latency of
  // epilogue-bound (short-K) tiles
  return EPI == Epi::kAdamW || SW_EPI_WG2 ? 384 : NUM_THREADS;
}
template <Epi EPI>
constexpr int p_stages() {
  return EPI == Epi::kAdamW ? (227 * 1024 - 1024 - 256 - OPT_SMEM) / P_STAGE_BYTES < 6
                                  ? (227 * 1024 - 1024 - 256 - OPT_SMEM) / P_STAGE_BYTES
                                  : 6
                            : 6;
}
template <Epi EPI>
constexpr int p_smem_bytes() {
  return p_stages<EPI>() * P_STAGE_BYTES + (EPI == Epi::kAdamW ? OPT_SMEM : 0) +
         (tma_epi<EPI>() ? 4 * 2 * EPI_TMA_BUF : 0) + 1024 + 256;
}

// fp32 tensor maps over p, m, v ([M, ldc], box OC columns x 32 rows, swizzle span = one row).
struct OptMaps {
  CUtensorMap p, m, v;
  CUtensorMap c;  // the output, for the TMA-store epilogue (kStoreF32 / kStoreBf16 / kResidF32)
  CUtensorMap a;   // kResidF32: the residual addend; kGeluBwd: the bf16 pre-activations; kBf16Delta: O
  CUtensorMap c2;  // kBiasGelu: the activation output
};



// AdamW on one warp's 32 rows x OC columns with p/m/v resident in shared memory (TMA swizzled
// rows: 16-byte chunk c of row r sits at chunk c ^ (r & 7) for 128-byte rows, c ^ ((r >> 1) & 3)
// for 64-byte rows). Lane = row, so the gradient row comes straight from the tcgen05.ld
// registers; rows/columns outside the matrix were zero-filled by TMA and are clipped by the TMA
// store, so only the bf16 shadow store is masked.
__device__ __forceinline__ int opt_pos(int r, int c) {
  return OC == 32 ? (r * 8 + (c ^ (r & 7))) : (r * 4 + (c ^ ((r >> 1) & 3)));
}

__device__ __forceinline__ void adamw_chunk_smem(const GemmParams& p, float* sbox, int row, int col0, int ncols,
                                                 const uint32_t* r, uint32_t lane) {
  float4* sp = reinterpret_cast<float4*>(sbox);
  float4* sm = reinterpret_cast<float4*>(sbox + OPT_ARR / 4);
  float4* sv = reinterpret_cast<float4*>(sbox + OPT_ARR / 2);
  const float y1 = dev::rcp_refined(p.adam_c1), y2 = dev::rcp_refined(p.adam_c2);
  const bool fast = p.adam_fast != 0;
  const int L = static_cast<int>(lane);
  bool bad = false;
  uint32_t slow = 0;
  float4 pv[OC / 4];
  // a non-finite loss (or an earlier non-finite gradient) gates the update: the staged p/m/v
  // go back unchanged (the caller's TMA store rewrites the same bytes) and the shadow is kept
  if (__ldcg(p.adam_flag) != 0) return;
#pragma unroll
  for (int c = 0; c < OC / 4; ++c) {
    const int at = opt_pos(L, c);
    float4 P = sp[at], M = sm[at], V = sv[at];
    const float g0 = __uint_as_float(r[4 * c]) * p.alpha, g1 = __uint_as_float(r[4 * c + 1]) * p.alpha;
    const float g2 = __uint_as_float(r[4 * c + 2]) * p.alpha, g3 = __uint_as_float(r[4 * c + 3]) * p.alpha;
    bad |= !(isfinite(g0) & isfinite(g1) & isfinite(g2) & isfinite(g3));
    slow |= fast && dev::adamw_update_fast(P.x, M.x, V.x, g0, p.adam_lr, p.adam_b1, p.adam_b2, p.adam_eps, p.adam_wd, p.adam_c1, p.adam_c2, y1, y2) ? 0u : 1u << (4 * c);
    slow |= fast && dev::adamw_update_fast(P.y, M.y, V.y, g1, p.adam_lr, p.adam_b1, p.adam_b2, p.adam_eps, p.adam_wd, p.adam_c1, p.adam_c2, y1, y2) ? 0u : 1u << (4 * c + 1);
    slow |= fast && dev::adamw_update_fast(P.z, M.z, V.z, g2, p.adam_lr, p.adam_b1, p.adam_b2, p.adam_eps, p.adam_wd, p.adam_c1, p.adam_c2, y1, y2) ? 0u : 1u << (4 * c + 2);
    slow |= fast && dev::adamw_update_fast(P.w, M.w, V.w, g3, p.adam_lr, p.adam_b1, p.adam_b2, p.adam_eps, p.adam_wd, p.adam_c1, p.adam_c2, y1, y2) ? 0u : 1u << (4 * c + 3);
    sp[at] = P;
    sm[at] = M;
    sv[at] = V;
    pv[c] = P;
  }
  if (__any_sync(0xffffffffu, slow != 0)) {
    // IEEE fallback for the elements whose intermediates left the fast-path range (their p/m/v
    // in shared memory are still the old values)
#pragma unroll
    for (int c = 0; c < OC / 4; ++c) {
      if ((slow >> (4 * c)) & 0xfu) {
        const int at = opt_pos(L, c);
        float4 P = sp[at], M = sm[at], V = sv[at];
        if (slow & (1u << (4 * c))) dev::adamw_update(P.x, M.x, V.x, __uint_as_float(r[4 * c]) * p.alpha, p.adam_lr, p.adam_b1, p.adam_b2, p.adam_eps, p.adam_wd, p.adam_c1, p.adam_c2);
        if (slow & (1u << (4 * c + 1))) dev::adamw_update(P.y, M.y, V.y, __uint_as_float(r[4 * c + 1]) * p.alpha, p.adam_lr, p.adam_b1, p.adam_b2, p.adam_eps, p.adam_wd, p.adam_c1, p.adam_c2);
        if (slow & (1u << (4 * c + 2))) dev::adamw_update(P.z, M.z, V.z, __uint_as_float(r[4 * c + 2]) * p.alpha, p.adam_lr, p.adam_b1, p.adam_b2, p.adam_eps, p.adam_wd, p.adam_c1, p.adam_c2);
        if (slow & (1u << (4 * c + 3))) dev::adamw_update(P.w, M.w, V.w, __uint_as_float(r[4 * c + 3]) * p.alpha, p.adam_lr, p.adam_b1, p.adam_b2, p.adam_eps, p.adam_wd, p.adam_c1, p.adam_c2);
        sp[at] = P;
        sm[at] = M;
        sv[at] = V;
        pv[c] = P;
      }
    }
  }
  if (row < p.M && !SW_EXP_NO_SHADOW_STORE) {  // (the macro: timing experiment only)
    __nv_bfloat16* w = reinterpret_cast<__nv_bfloat16*>(p.adam_w) + static_cast<int64_t>(row) * p.ldc + col0;
#pragma unroll
    for (int c = 0; c < OC / 4; c += 2) {
      if (4 * c < ncols) {
        uint4 o;
        o.x = dev::pack_bf16x2(pv[c].x, pv[c].y);
        o.y = dev::pack_bf16x2(pv[c].z, pv[c].w);
        o.z = dev::pack_bf16x2(pv[c + 1].x, pv[c + 1].y);
        o.w = dev::pack_bf16x2(pv[c + 1].z, pv[c + 1].w);
        *reinterpret_cast<uint4*>(w + 4 * c) = o;
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(p.adam_flag, 1);
}

// Phase trace of one CTA (tools/gemm_trace.py), per tile i < 64 of that CTA:
// [8i] MMA passed tempty, [8i+1] MMA issued the last k-block, [8i+2] cycles the MMA warp waited
// on full[] in the tile, [8i+3] epilogue warp 4 passed tfull, [8i+4] warp 4 released the
// accumulator, [8i+5] warp 8 released it, [8i+6] cycles warp 4 waited on ofull in the tile.
__device__ unsigned long long g_gemm_trace[1024];

template <Epi EPI>
__global__ void __cluster_dims__(GEMM_CL, 1, 1) __launch_bounds__(p_threads<EPI>(), 1)
    gemm_bf16_2sm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ OptMaps om, const GemmParams p) {
  constexpr int P_STAGES = p_stages<EPI>();
  constexpr bool kOpt = EPI == Epi::kAdamW;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + P_STAGES * P_A_STAGE;
  uint8_t* sOpt = sB + P_STAGES * P_B_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sOpt + (kOpt ? OPT_SMEM : 0) + (tma_epi<EPI>() ? 4 * 2 * EPI_TMA_BUF : 0));
  uint64_t* empty = full + P_STAGES;
  uint64_t* tfull = empty + P_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* ofull = tempty + 2;
  uint64_t* oempty = ofull + 3;
  uint64_t* eload = oempty + 3;  // [4 warps][2 buffers] residual-chunk loads (TMA epilogue)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(eload + 8);

  const uint32_t warp = dev::warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  // cluster = GEMM_CL / 2 CTA pairs on one tile row: pair pidx of the cluster takes n-block
  // 2 nbp + pidx of cluster tile (mb, nbp), and with GEMM_CL == 4 the two CTAs holding the same
  // A rows (ranks prank and prank + 2) each fetch half of them and multicast it to both
  const uint32_t crank = dev::cluster_ctarank();
  const uint32_t rank = crank & 1u;   // rank inside the CTA pair
  const int pidx = static_cast<int>(crank >> 1);

  const int num_m = (p.M + 2 * BM - 1) / (2 * BM);  // pair tiles along M (256 rows)
  constexpr bool kGlu = EPI == Epi::kSwiGLU;
  const int num_n = kGlu ? (p.N + 127) / 128 : (p.N + BN - 1) / BN;  // SwiGLU: 128 h columns per tile
  const int num_tiles = num_m * num_n;
  const int num_kb = (p.K + BK - 1) / BK;
  const int pair = static_cast<int>(blockIdx.x) / GEMM_CL;     // cluster index
  const int npairs = static_cast<int>(gridDim.x) / GEMM_CL;
  const int num_nc = GEMM_CL == 4 ? (num_n + 1) / 2 : num_n;   // n-block units per cluster tile
  // split-K (kStoreF32): unit u is K slice u % nsplit of tile u / nsplit, so a tile's slices run
  // side by side and meet in C through TMA reduce-adds
  const int nsplit = p.split_k > 1 ? p.split_k : 1;
  const int num_units = num_m * num_nc * nsplit;
  auto pair_tile = [&](int u, int& mb, int& nb) {
    const int t = u / nsplit;
    if constexpr (GEMM_CL == 4) {
      int nbp;
      tile_coords(t, num_m, num_nc, mb, nbp);
      nb = 2 * nbp + pidx;  // past num_n on an odd tail: B reads zeros, the epilogue stores nothing
    } else {
      tile_coords(t, num_m, num_n, mb, nb);
    }
  };
  auto kb_lo = [&](int u) { return (u % nsplit) * num_kb / nsplit; };
  auto kb_hi = [&](int u) { return (u % nsplit + 1) * num_kb / nsplit; };

  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&tmA);
    dev::tma_prefetch_desc(&tmB);
    for (int s = 0; s < P_STAGES; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], GEMM_CL / 2);  // one MMA commit per pair of the cluster
    }
    for (int a = 0; a < 2; ++a) {
      dev::mbar_init(&tfull[a], 1);
      dev::mbar_init(&tempty[a], kOpt || SW_EPI_WG2 ? 16 : 8);  // epilogue warps of both CTAs
    }
    for (int a = 0; a < 8; ++a) dev::mbar_init(&eload[a], 1);
    for (int a = 0; a < OPT_NBUF; ++a) {
      dev::mbar_init(&ofull[a], 1);
      dev::mbar_init(&oempty[a], 4);
    }
    dev::fence_barrier_init();
  }
  if (warp == 2) dev::tmem_alloc_2sm<TMEM_COLS>(tmem_slot);
  dev::tc_fence_before();
  dev::cluster_sync();
  dev::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < num_units; t += npairs) {
        int mb, nb;
        pair_tile(t, mb, nb);
        const int m0 = mb * 2 * BM + static_cast<int>(rank) * BM;
        // SwiGLU: CTA 0 stages the tile's 128 gate rows, CTA 1 the matching 128 up rows
        const int n0 = kGlu ? (rank == 0 ? nb * 128 : p.swiglu_half + nb * 128)
                            : nb * BN + static_cast<int>(rank) * 128;
        for (int kb = kb_lo(t), kb_end = kb_hi(t); kb < kb_end; ++kb) {
          dev::mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) dev::mbar_arrive_expect_tx(&full[stage], 2 * P_STAGE_BYTES);
          const int k0 = kb * BK;
          uint8_t* a_dst = sA + stage * P_A_STAGE;
          uint8_t* b_dst = sB + stage * P_B_STAGE;
          if constexpr (GEMM_CL == 4) {
            // 64 of the 128 A rows (K-major: one [64 k x 64 rows] box; MN-major: one of the two
            // [64 rows x 64 k] boxes), landing in both CTAs that hold these rows
            const uint16_t mc = static_cast<uint16_t>((1u << rank) | (1u << (rank + 2)));
            if (!p.a_mn_major) {
              dev::tma_load_2d_2sm_mc(a_dst + pidx * 8192, &tmA, &full[stage], k0, m0 + 64 * pidx, mc);
            } else {
              dev::tma_load_2d_2sm_mc(a_dst + pidx * 8192, &tmA, &full[stage], m0 + 64 * pidx, k0, mc);
            }
          } else if (!p.a_mn_major) {
            dev::tma_load_2d_2sm(a_dst, &tmA, &full[stage], k0, m0);
          } else {
            dev::tma_load_2d_2sm(a_dst, &tmA, &full[stage], m0, k0);
            dev::tma_load_2d_2sm(a_dst + 8192, &tmA, &full[stage], m0 + 64, k0);
          }
          if (!p.b_mn_major) {
            dev::tma_load_2d_2sm(b_dst, &tmB, &full[stage], k0, n0);
          } else {
            dev::tma_load_2d_2sm(b_dst, &tmB, &full[stage], n0, k0);
            dev::tma_load_2d_2sm(b_dst + 8192, &tmB, &full[stage], n0 + 64, k0);
          }
          if (++stage == P_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // the whole warp runs the issue loop (converged: descriptors stay in uniform registers);
      // one elected lane issues the MMAs and commits
      const uint32_t idesc = dev::make_idesc_bf16(2 * BM, BN, p.a_mn_major, p.b_mn_major);
      const uint64_t a0 = p.a_mn_major ? dev::make_sdesc_sw128(dev::smem_u32(sA), 8192, 1024)
                                       : dev::make_sdesc_sw128(dev::smem_u32(sA), 16, 1024);
      const uint64_t b0 = p.b_mn_major ? dev::make_sdesc_sw128(dev::smem_u32(sB), 8192, 1024)
                                       : dev::make_sdesc_sw128(dev::smem_u32(sB), 16, 1024);
      const uint64_t a_step = p.a_mn_major ? (2048 >> 4) : (32 >> 4);  // per 16-deep k step
      const uint64_t b_step = p.b_mn_major ? (2048 >> 4) : (32 >> 4);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const bool tr = static_cast<int>(blockIdx.x) == p.trace_cta;
      int ti = 0;
      for (int t = pair; t < num_units; t += npairs, ++ti) {
        dev::mbar_wait(&tempty[acc], acc_phase ^ 1);
        dev::tc_fence_after();
        if (tr && lane == 0 && ti < 64) g_gemm_trace[8 * ti] = clock64();
        long long waited = 0;
        const uint32_t d_tmem = tmem_base + acc * BN;
        const int kb0 = kb_lo(t);
        for (int kb = kb0, kb_end = kb_hi(t); kb < kb_end; ++kb) {
          const long long w0 = tr ? clock64() : 0;
          dev::mbar_wait(&full[stage], phase);
          dev::tc_fence_after();
          if (tr) waited += clock64() - w0;
          const uint64_t as = a0 + static_cast<uint64_t>(stage * (P_A_STAGE >> 4));
          const uint64_t bs = b0 + static_cast<uint64_t>(stage * (P_B_STAGE >> 4));
          if (dev::elect_one_sync()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              dev::umma_f16_ss_2sm(d_tmem, as + k * a_step, bs + k * b_step, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
            // the stage is free once every pair that reads or multicasts into it is done
            dev::umma_commit_2sm(&empty[stage], GEMM_CL == 4 ? 0xF : 0x3);
          }
          __syncwarp();
          if (++stage == P_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (dev::elect_one_sync()) dev::umma_commit_2sm(&tfull[acc], static_cast<uint16_t>(0x3u << (2 * pidx)));
        __syncwarp();
        if (tr && lane == 0 && ti < 64) {
          g_gemm_trace[8 * ti + 1] = clock64();
          g_gemm_trace[8 * ti + 2] = waited;
        }
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp == 3) {
    if constexpr (kOpt && !SW_ADAMW_DIRECT) {
      if (lane == 0) {
        // ---------------- optimizer-state producer (TMA, one chunk ahead) ----------------
        dev::tma_prefetch_desc(&om.p);
        dev::tma_prefetch_desc(&om.m);
        dev::tma_prefetch_desc(&om.v);
        uint32_t uses[OPT_NBUF] = {0, 0};
        for (int t = pair; t < num_units; t += npairs) {
          int mb, nb;
          pair_tile(t, mb, nb);
          const int r0 = mb * 2 * BM + static_cast<int>(rank) * BM;
          const int n_left = p.N - nb * BN;
          // chunk c of the tile goes to buffer c & 1, i.e. to epilogue warpgroup c & 1
          for (int c = 0; c < BN / OC && c * OC < n_left; ++c) {
            const int buf = c & 1;
            dev::mbar_wait(&oempty[buf], (uses[buf] & 1) ^ 1);
            ++uses[buf];
#if SW_EXP_NO_STATE_LOAD  // timing experiment only (results invalid when set)
            dev::mbar_arrive(&ofull[buf]);
            continue;
#endif
            dev::mbar_arrive_expect_tx(&ofull[buf], OPT_BUF);
            uint8_t* dst = sOpt + buf * OPT_BUF;
            const int c0 = nb * BN + c * OC;
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              dev::tma_load_2d(dst + w * OPT_WBOX, &om.p, &ofull[buf], c0, r0 + 32 * w);
              dev::tma_load_2d(dst + OPT_ARR + w * OPT_WBOX, &om.m, &ofull[buf], c0, r0 + 32 * w);
              dev::tma_load_2d(dst + 2 * OPT_ARR + w * OPT_WBOX, &om.v, &ofull[buf], c0, r0 + 32 * w);
            }
          }
        }
      }
    }
  } else if (kOpt && SW_ADAMW_DIRECT && warp >= 4) {
    // ---------------- AdamW epilogue, direct: two warpgroups on alternate 32-column chunks ----------------
    const uint32_t q = warp & 3;
    const int wg = (static_cast<int>(warp) - 4) >> 2;
    float4* stage = reinterpret_cast<float4*>(sOpt) + (static_cast<int>(warp) - 4) * 256;
    const uint32_t tempty_leader = dev::mapa_shared(dev::smem_u32(&tempty[0]), crank & ~1u);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = pair; t < num_units; t += npairs) {
      int mb, nb;
      pair_tile(t, mb, nb);
      const int row0 = mb * 2 * BM + static_cast<int>(rank) * BM + static_cast<int>(q) * 32;
      dev::mbar_wait(&tfull[acc], acc_phase);
      dev::tc_fence_after();
#pragma unroll 1
      for (int j = wg; j < BN / 32; j += 2) {
        const int col0 = nb * BN + j * 32;
        if (col0 >= p.N) break;
        uint32_t r[32];
        dev::tmem_ld_32x32b_x32(tmem_base + ((q * 32) << 16) + acc * BN + j * 32, r);
        dev::tmem_ld_wait();
        adamw_chunk(p, stage, row0, col0, min(32, p.N - col0), r, lane);
      }
      dev::tc_fence_before();
      if (lane == 0) dev::mbar_arrive_cluster(tempty_leader + acc * 8);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (kOpt && warp >= 4) {
    // ---------------- AdamW epilogue: two warpgroups on alternate 16-column chunks ----------------
    // Warpgroup wg (warps 4-7 / 8-11, the same TMEM lane quarters) owns chunks c = 2j + wg and
    // the state buffer wg: one chunk per warpgroup in flight, so the latency-bound update of
    // one overlaps the other's loads, math and TMA stores.
    const uint32_t q = warp & 3;
    const int wg = (static_cast<int>(warp) - 4) >> 2;
    const uint32_t tempty_leader = dev::mapa_shared(dev::smem_u32(&tempty[0]), crank & ~1u);
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t uses = 0;
    const bool tr = static_cast<int>(blockIdx.x) == p.trace_cta && lane == 0;
    int ti = 0;
    for (int t = pair; t < num_units; t += npairs, ++ti) {
      int mb, nb;
      pair_tile(t, mb, nb);
      const int row = mb * 2 * BM + static_cast<int>(rank) * BM + static_cast<int>(q) * 32 + static_cast<int>(lane);
      dev::mbar_wait(&tfull[acc], acc_phase);
      dev::tc_fence_after();
      if (tr && warp == 4 && ti < 64) g_gemm_trace[8 * ti + 3] = clock64();
      long long owait = 0;
#pragma unroll 1
      for (int j = 0; j < BN / (2 * OC); ++j) {
        const int col0 = nb * BN + (2 * j + wg) * OC;
        if (col0 >= p.N) break;
        uint32_t r[OC];
        dev::tmem_ld_32x32b_x16(tmem_base + ((q * 32) << 16) + acc * BN + (2 * j + wg) * OC, r);
        dev::tmem_ld_wait();
        const long long o0 = tr ? clock64() : 0;
        dev::mbar_wait(&ofull[wg], uses & 1);
        if (tr) owait += clock64() - o0;
        ++uses;
        float* sbox = reinterpret_cast<float*>(sOpt + wg * OPT_BUF) + q * (OPT_WBOX / 4);
        adamw_chunk_smem(p, sbox, row, col0, min(OC, p.N - col0), r, lane);
        dev::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const int rw = row - static_cast<int>(lane);
#if !SW_EXP_NO_STATE_STORE  // timing experiment only (results invalid when set)
          dev::tma_store_2d(&om.p, sbox, col0, rw);
          dev::tma_store_2d(&om.m, sbox + OPT_ARR / 4, col0, rw);
          dev::tma_store_2d(&om.v, sbox + OPT_ARR / 2, col0, rw);
#endif
          dev::bulk_commit();
          dev::bulk_wait_read();  // the stores have left shared memory: hand the buffer back
          dev::mbar_arrive(&oempty[wg]);
        }
      }
      dev::tc_fence_before();
      if (tr && (warp == 4 || warp == 8) && ti < 64) {
        g_gemm_trace[8 * ti + (warp == 4 ? 4 : 5)] = clock64();
        if (warp == 4) g_gemm_trace[8 * ti + 6] = owait;
      }
      if (lane == 0) dev::mbar_arrive_cluster(tempty_leader + acc * 8);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    const uint32_t q = warp & 3;
    // chunk stride and first chunk of this warp's warpgroup (one warpgroup: every chunk)
    const int cstep = SW_EPI_WG2 ? 2 : 1, cfirst = SW_EPI_WG2 ? (static_cast<int>(warp) - 4) >> 2 : 0;
    uint32_t rphase[2] = {0u, 0u};  // TMA residual-load barrier phases of the two staging buffers
    (void)rphase;
    const uint32_t tempty_leader = dev::mapa_shared(dev::smem_u32(&tempty[0]), crank & ~1u);
    int acc = 0;
    uint32_t acc_phase = 0;
    const bool tr = static_cast<int>(blockIdx.x) == p.trace_cta && lane == 0 && warp == 4;
    int ti = 0;
    for (int t = pair; t < num_units; t += npairs, ++ti) {
      int mb, nb;
      pair_tile(t, mb, nb);
      const int row = mb * 2 * BM + static_cast<int>(rank) * BM + static_cast<int>(q) * 32 + static_cast<int>(lane);
      dev::mbar_wait(&tfull[acc], acc_phase);
      dev::tc_fence_after();
      if (tr && ti < 64) g_gemm_trace[8 * ti + 3] = clock64();
      const int n_left = p.N - nb * BN;
      if constexpr (kGlu) {
        // accumulator columns [0,128) = gate, [128,256) = up for h columns nb*128 + [0,128)
        const int h_left = p.N - nb * 128;
#pragma unroll 1
        for (int j = cfirst; j < 4; j += cstep) {
          const int ncols = min(32, h_left - j * 32);
          if (ncols <= 0) break;
          uint32_t rg[32], ru[32];
          dev::tmem_ld_32x32b_x32(tmem_base + ((q * 32) << 16) + acc * BN + j * 32, rg);
          dev::tmem_ld_32x32b_x32(tmem_base + ((q * 32) << 16) + acc * BN + 128 + j * 32, ru);
          dev::tmem_ld_wait();
          if (row < p.M) {
            const int c0 = nb * 128 + j * 32;
            __nv_bfloat16* hrow = reinterpret_cast<__nv_bfloat16*>(p.C) + static_cast<int64_t>(row) * p.ldc + c0;
            __nv_bfloat16* prow = reinterpret_cast<__nv_bfloat16*>(p.C2) + static_cast<int64_t>(row) * p.ldc2 + c0;
#pragma unroll
            for (int c = 0; c < 32; c += 8) {
              if (c < ncols) {
                uint32_t hw[4], gw[4], uw[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  // the stored bf16 pre-activations are what the backward differentiates
                  const float2 g = dev::unpack_bf16x2(
                      dev::pack_bf16x2(__uint_as_float(rg[c + 2 * e]), __uint_as_float(rg[c + 2 * e + 1])));
                  const float2 u = dev::unpack_bf16x2(
                      dev::pack_bf16x2(__uint_as_float(ru[c + 2 * e]), __uint_as_float(ru[c + 2 * e + 1])));
                  gw[e] = dev::pack_bf16x2(g.x, g.y);
                  uw[e] = dev::pack_bf16x2(u.x, u.y);
                  hw[e] = dev::pack_bf16x2(dev::silu(g.x) * u.x, dev::silu(g.y) * u.y);
                }
                *reinterpret_cast<uint4*>(hrow + c) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                *reinterpret_cast<uint4*>(prow + c) = make_uint4(gw[0], gw[1], gw[2], gw[3]);
                *reinterpret_cast<uint4*>(prow + p.swiglu_half + c) = make_uint4(uw[0], uw[1], uw[2], uw[3]);
              }
            }
          }
        }
      }
#pragma unroll 1
#if SW_EPI_PF == 0
      if constexpr (tma_epi<EPI>()) {
        if (!p.accumulate || nsplit > 1) {
          // stage in shared memory (lane = row of the warp's 32, swizzled 16-byte units), one TMA
          // store per chunk (a reduce-add under split-K); a buffer is rewritten only after its
          // previous store read it
          uint8_t* stg = sOpt + (static_cast<int>(warp) - 4) * 2 * EPI_TMA_BUF;
          constexpr bool f32 = EPI == Epi::kStoreF32 || EPI == Epi::kResidF32;
          constexpr bool resid = EPI == Epi::kResidF32, gbwd = EPI == Epi::kGeluBwd, gfwd = EPI == Epi::kBiasGelu;
          constexpr bool dlt = EPI == Epi::kBf16Delta;
          float dsum = 0.f;  // kBf16Delta: this row's dO . O over the current 128-column head
          constexpr int chunk_bytes = f32 ? 4096 : 2048;
#pragma unroll 1
          for (int j = 0; j < BN / 32; ++j) {
            if (j * 32 >= n_left) break;
            uint64_t* ebar = &eload[(static_cast<int>(warp) - 4) * 2 + (j & 1)];
            if (lane == 0) {
              dev::bulk_wait_read_1();  // buffer (j & 1) was read by the store two chunks back
              if constexpr (resid || gbwd || dlt) {  // the addend / pre-activation chunk lands while the accumulator is read
                dev::mbar_arrive_expect_tx(ebar, chunk_bytes);
                dev::tma_load_2d(stg + (j & 1) * EPI_TMA_BUF, &om.a, ebar, nb * BN + j * 32, row - static_cast<int>(lane));
              }
            }
            uint32_t r[32];
            dev::tmem_ld_32x32b_x32(tmem_base + ((q * 32) << 16) + acc * BN + j * 32, r);
            dev::tmem_ld_wait();
            float v[32];
            epilogue_values(p, nb * BN + j * 32, min(32, n_left - j * 32), r, v);
            if constexpr (EPI == Epi::kStoreBf16) {
              if (p.relu) {
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
              }
            }
            __syncwarp();
            uint8_t* buf = stg + (j & 1) * EPI_TMA_BUF + lane * (f32 ? 128 : 64);
            if constexpr (resid) {
              dev::mbar_wait(ebar, rphase[j & 1]);
              rphase[j & 1] ^= 1u;
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                float4* pa = reinterpret_cast<float4*>(buf + ((u ^ (lane & 7)) << 4));
                const float4 a = *pa;
                *pa = make_float4(v[4 * u] + a.x, v[4 * u + 1] + a.y, v[4 * u + 2] + a.z, v[4 * u + 3] + a.w);
              }
            } else if constexpr (gbwd) {  // dpre = acc * gelu'(pre), in place over the loaded pre chunk
              dev::mbar_wait(ebar, rphase[j & 1]);
              rphase[j & 1] ^= 1u;
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                uint4* pa = reinterpret_cast<uint4*>(buf + ((u ^ ((lane >> 1) & 3)) << 4));
                const uint4 raw = *pa;
                const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
                uint32_t o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 x = dev::unpack_bf16x2(w[e]);
                  o[e] = dev::pack_bf16x2(v[8 * u + 2 * e] * act_grad(p, x.x),
                                          v[8 * u + 2 * e + 1] * act_grad(p, x.y));
                }
                *pa = make_uint4(o[0], o[1], o[2], o[3]);
              }
            } else if constexpr (dlt) {  // dO (bf16) in place over the loaded O chunk; dO . O into dsum
              dev::mbar_wait(ebar, rphase[j & 1]);
              rphase[j & 1] ^= 1u;
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                uint4* pa = reinterpret_cast<uint4*>(buf + ((u ^ ((lane >> 1) & 3)) << 4));
                const uint4 raw = *pa;
                const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
                uint32_t o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  o[e] = dev::pack_bf16x2(v[8 * u + 2 * e], v[8 * u + 2 * e + 1]);
                  const float2 x = dev::unpack_bf16x2(w[e]), y = dev::unpack_bf16x2(o[e]);
                  dsum = fmaf(x.x, y.x, fmaf(x.y, y.y, dsum));
                }
                *pa = make_uint4(o[0], o[1], o[2], o[3]);
              }
              if ((j & 3) == 3) {
                const int col = nb * BN + j * 32;
                if (row < p.M) {
                  const int b = row / p.delta_T, t = row - b * p.delta_T;
                  p.delta[(static_cast<int64_t>(b) * (p.N >> 7) + (col >> 7)) * p.delta_T + t] = dsum;
                }
                dsum = 0.f;
              }
            } else if constexpr (gfwd) {  // pre-activation in the first half, gelu in the second
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int sw = (u ^ ((lane >> 1) & 3)) << 4;
                *reinterpret_cast<uint4*>(buf + sw) =
                    make_uint4(dev::pack_bf16x2(v[8 * u], v[8 * u + 1]), dev::pack_bf16x2(v[8 * u + 2], v[8 * u + 3]),
                               dev::pack_bf16x2(v[8 * u + 4], v[8 * u + 5]), dev::pack_bf16x2(v[8 * u + 6], v[8 * u + 7]));
                *reinterpret_cast<uint4*>(buf + 2048 + sw) =
                    make_uint4(dev::pack_bf16x2(dev::gelu_tanh(v[8 * u]), dev::gelu_tanh(v[8 * u + 1])),
                               dev::pack_bf16x2(dev::gelu_tanh(v[8 * u + 2]), dev::gelu_tanh(v[8 * u + 3])),
                               dev::pack_bf16x2(dev::gelu_tanh(v[8 * u + 4]), dev::gelu_tanh(v[8 * u + 5])),
                               dev::pack_bf16x2(dev::gelu_tanh(v[8 * u + 6]), dev::gelu_tanh(v[8 * u + 7])));
              }
            } else if constexpr (f32) {
#pragma unroll
              for (int u = 0; u < 8; ++u)
                *reinterpret_cast<float4*>(buf + ((u ^ (lane & 7)) << 4)) =
                    make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                *reinterpret_cast<uint4*>(buf + ((u ^ ((lane >> 1) & 3)) << 4)) =
                    make_uint4(dev::pack_bf16x2(v[8 * u], v[8 * u + 1]), dev::pack_bf16x2(v[8 * u + 2], v[8 * u + 3]),
                               dev::pack_bf16x2(v[8 * u + 4], v[8 * u + 5]), dev::pack_bf16x2(v[8 * u + 6], v[8 * u + 7]));
            }
            dev::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (nsplit > 1) {
                dev::tma_reduce_add_2d(&om.c, stg + (j & 1) * EPI_TMA_BUF, nb * BN + j * 32, row - static_cast<int>(lane));
              } else {
                dev::tma_store_2d(&om.c, stg + (j & 1) * EPI_TMA_BUF, nb * BN + j * 32, row - static_cast<int>(lane));
              }
              if constexpr (gfwd)
                dev::tma_store_2d(&om.c2, stg + (j & 1) * EPI_TMA_BUF + 2048, nb * BN + j * 32,
                                  row - static_cast<int>(lane));
              dev::bulk_commit();
            }
            if constexpr (gbwd) {
              if (p.colsum != nullptr) {
                // column sums of the stored chunk (the bias gradient): lanes 0-15 take the even rows,
                // 16-31 the odd ones, lane l % 16 owns columns 2(l % 16) and 2(l % 16) + 1
                const uint8_t* cb = stg + (j & 1) * EPI_TMA_BUF;
                const int cl = static_cast<int>(lane & 15), rh = static_cast<int>(lane >> 4);
                float s0 = 0.f, s1 = 0.f;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                  const int rr = 2 * i + rh;
                  const float2 x = dev::unpack_bf16x2(*reinterpret_cast<const uint32_t*>(
                      cb + rr * 64 + (((cl >> 2) ^ ((rr >> 1) & 3)) << 4) + (cl & 3) * 4));
                  s0 += x.x;
                  s1 += x.y;
                }
                s0 += __shfl_down_sync(0xffffffffu, s0, 16);
                s1 += __shfl_down_sync(0xffffffffu, s1, 16);
                const int col = nb * BN + j * 32 + 2 * cl;
                const int rb = row - static_cast<int>(lane);
                if (lane < 16 && rb < p.M && col < p.N)
                  *reinterpret_cast<float2*>(p.colsum + static_cast<int64_t>(rb >> 5) * p.N + col) =
                      make_float2(s0, s1);
              }
            }
          }
        } else {
#pragma unroll 1
          for (int j = 0; j < BN / 32; ++j) {
            const int ncols = min(32, n_left - j * 32);
            if (ncols <= 0) break;
            uint32_t r[32];
            dev::tmem_ld_32x32b_x32(tmem_base + ((q * 32) << 16) + acc * BN + j * 32, r);
            dev::tmem_ld_wait();
            if (row < p.M) epilogue_chunk<EPI>(p, row, nb * BN + j * 32, ncols, r);
          }
        }
      } else {
#pragma unroll 1
      for (int j = cfirst; j < (kGlu ? 0 : BN / 32); j += cstep) {
        const int ncols = min(32, n_left - j * 32);
        if (ncols <= 0) break;
        uint32_t r[32];
        dev::tmem_ld_32x32b_x32(tmem_base + ((q * 32) << 16) + acc * BN + j * 32, r);
        dev::tmem_ld_wait();
        if (row < p.M) epilogue_chunk<EPI>(p, row, nb * BN + j * 32, ncols, r);
      }
      }
#else
      if constexpr (!kGlu) {
        // the next chunk's tcgen05.ld is in flight while this one is processed
        const int nch = min(BN / 32, (n_left + 31) / 32);
        // (two register buffers, the loop unrolled by two only: the GeLU epilogues are long)
        uint32_t r0[32], r1[32];
        const uint32_t tbase = tmem_base + ((q * 32) << 16) + acc * BN;
        dev::tmem_ld_32x32b_x32(tbase, r0);
        dev::tmem_ld_wait();
#pragma unroll 1
        for (int j = 0; j < nch; j += 2) {
          if (j + 1 < nch) dev::tmem_ld_32x32b_x32(tbase + (j + 1) * 32, r1);
          if (row < p.M) epilogue_chunk<EPI>(p, row, nb * BN + j * 32, min(32, n_left - j * 32), r0);
          dev::tmem_ld_wait();
          if (j + 1 < nch) {
            if (j + 2 < nch) dev::tmem_ld_32x32b_x32(tbase + (j + 2) * 32, r0);
            if (row < p.M) epilogue_chunk<EPI>(p, row, nb * BN + (j + 1) * 32, min(32, n_left - (j + 1) * 32), r1);
            dev::tmem_ld_wait();
          }
        }
      }
#endif
      dev::tc_fence_before();
      if (tr && ti < 64) g_gemm_trace[8 * ti + 4] = clock64();
      if (lane == 0) dev::mbar_arrive_cluster(tempty_leader + acc * 8);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  if constexpr ((kOpt && !SW_ADAMW_DIRECT) || tma_epi<EPI>()) {
    if (warp >= 4 && lane == 0) dev::bulk_wait_all();
  }
  dev::tc_fence_before();
  dev::cluster_sync();
  if (warp == 2) {
    dev::tc_fence_after();
    dev::tmem_dealloc_2sm<TMEM_COLS>(tmem_base);
  }
}

template <Epi EPI>
cudaError_t launch_2sm(const GemmParams& p, cudaStream_t stream) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_2sm_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         p_smem_bytes<EPI>());
    if (e != cudaSuccess) return e;
    configured = true;
  }
  // K-major A: one [64 k x 128 rows] box per stage, or half of it per multicasting CTA
  CUtensorMap ta = p.a_mn_major ? make_tmap_bf16_2d(p.A, p.M, p.K, p.lda, 64, 64)
                                : make_tmap_bf16_2d(p.A, p.K, p.M, p.lda, 64, GEMM_CL == 4 ? 64 : BM);
  const uint64_t b_rows = EPI == Epi::kSwiGLU ? 2ull * p.swiglu_half : static_cast<uint64_t>(p.N);
  CUtensorMap tb = p.b_mn_major ? make_tmap_bf16_2d(p.B, p.N, p.K, p.ldb, 64, 64)
                                : make_tmap_bf16_2d(p.B, p.K, b_rows, p.ldb, 64, 128);
  const int num_n = EPI == Epi::kSwiGLU ? (p.N + 127) / 128 : (p.N + BN - 1) / BN;
  const int num_units = ((p.M + 2 * BM - 1) / (2 * BM)) * (GEMM_CL == 4 ? (num_n + 1) / 2 : num_n) *
                        (p.split_k > 1 ? p.split_k : 1);
  const int sms = (p.num_sms > 0 ? p.num_sms : device_sm_count()) & ~(GEMM_CL - 1);
  const int grid = GEMM_CL * num_units < sms ? GEMM_CL * num_units : sms;
  OptMaps om{};
  if constexpr (tma_epi<EPI>()) {
    if (!p.accumulate || p.split_k > 1) {
      constexpr bool f32 = EPI == Epi::kStoreF32 || EPI == Epi::kResidF32;
      om.c = f32 ? make_tmap_f32_2d(p.C, p.N, p.M, p.ldc, 32, 32)
                 : make_tmap_bf16_2d_rowswz(p.C, p.N, p.M, p.ldc, 32, 32);
      if constexpr (EPI == Epi::kResidF32) om.a = make_tmap_f32_2d(p.aux, p.N, p.M, p.ld_aux, 32, 32);
      if constexpr (EPI == Epi::kGeluBwd || EPI == Epi::kBf16Delta)
        om.a = make_tmap_bf16_2d_rowswz(p.aux, p.N, p.M, p.ld_aux, 32, 32);
      if constexpr (EPI == Epi::kBiasGelu) om.c2 = make_tmap_bf16_2d_rowswz(p.C2, p.N, p.M, p.ldc2, 32, 32);
    }
  }
  if constexpr (EPI == Epi::kAdamW) {
    om.p = make_tmap_f32_2d(p.adam_p, p.N, p.M, p.ldc, OC, 32);
    om.m = make_tmap_f32_2d(p.adam_m, p.N, p.M, p.ldc, OC, 32);
    om.v = make_tmap_f32_2d(p.adam_v, p.N, p.M, p.ldc, OC, 32);
  }
  static const int trace_cta = [] {
    const char* e = std::getenv("SW_GEMM_TRACE_CTA");
    return e != nullptr ? std::atoi(e) : -1;
  }();
  GemmParams q = p;
  q.trace_cta = trace_cta;
  gemm_bf16_2sm_kernel<EPI><<<grid, p_threads<EPI>(), p_smem_bytes<EPI>(), stream>>>(ta, tb, om, q);
  return cudaGetLastError();
}

template <Epi EPI>
cudaError_t launch(const GemmParams& p, cudaStream_t stream) {
  if (use_pairs()) return launch_2sm<EPI>(p, stream);
  if constexpr (EPI == Epi::kSwiGLU) {
    throw std::runtime_error("gemm_bf16: the SwiGLU epilogue needs the CTA-pair kernel (unset SW_GEMM_1SM)");
  }
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_kernel<EPI>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  CUtensorMap ta = p.a_mn_major ? make_tmap_bf16_2d(p.A, p.M, p.K, p.lda, 64, 64)
                                : make_tmap_bf16_2d(p.A, p.K, p.M, p.lda, 64, BM);
  CUtensorMap tb = p.b_mn_major ? make_tmap_bf16_2d(p.B, p.N, p.K, p.ldb, 64, 64)
                                : make_tmap_bf16_2d(p.B, p.K, p.N, p.ldb, 64, BN);
  const int num_tiles = ((p.M + BM - 1) / BM) * ((p.N + BN - 1) / BN);
  const int sms = p.num_sms > 0 ? p.num_sms : device_sm_count();
  const int grid = num_tiles < sms ? num_tiles : sms;
  gemm_bf16_kernel<EPI><<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(ta, tb, p);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Small-M path (M <= 8, K-major operands): the decode step's GEMMs are weight-streaming GEMVs.
// One CTA per 16 output columns streams those weight rows once (16-byte streaming loads; each
// warp keeps two rows in flight) against the M activation rows (L1-resident), then hands the
// chunk of every row to the same epilogue as the tensor-core kernel. HBM-bound by design.
// ---------------------------------------------------------------------------------------------
constexpr int GEMV_MAX_M = 8;
#ifndef SW_GEMV_COLS
#define SW_GEMV_COLS 16  // >= 8 (16-byte bf16 stores in the epilogue)
#endif
constexpr int GEMV_COLS = SW_GEMV_COLS;  // output columns per CTA (enough CTAs to cover the SMs at N = d_model)

// KSPLIT warp octets split K (more loads in flight per CTA: the narrow N = d_model GEMVs have
// fewer CTAs than the HBM latency needs); UNROLL k-steps of weight loads in flight per warp.
template <Epi EPI, int GEMV_KSPLIT, int GEMV_UNROLL, int MX>
__global__ void __launch_bounds__(256 * GEMV_KSPLIT) gemv_bf16_kernel(const GemmParams p) {
  __shared__ float sout[GEMV_MAX_M][2 * GEMV_COLS];
  __shared__ float spart[GEMV_KSPLIT > 1 ? GEMV_KSPLIT - 1 : 1][2 * GEMV_COLS][MX];
  constexpr bool kGlu = EPI == Epi::kSwiGLU;
  constexpr int ROWS = kGlu ? 2 * GEMV_COLS : GEMV_COLS;  // SwiGLU: the gate rows and the matching up rows
  constexpr int RPW = ROWS / 8 > 0 ? ROWS / 8 : 1;         // weight rows per warp, streamed together
  const int K = p.K, M = p.M;
  const int c0 = blockIdx.x * GEMV_COLS;
  const int ks = static_cast<int>(threadIdx.x >> 8);  // K slice of this warp octet
  const int warp = (threadIdx.x >> 5) & 7, lane = threadIdx.x & 31;
  const __nv_bfloat16* w[RPW];
  bool ok[RPW];
#pragma unroll
  for (int j = 0; j < RPW; ++j) {
    const int rr = warp + 8 * j;
    const int col = c0 + (rr % GEMV_COLS);
    ok[j] = col < p.N;
    const int wrow = kGlu ? (rr < GEMV_COLS ? col : p.swiglu_half + col) : col;
    w[j] = reinterpret_cast<const __nv_bfloat16*>(p.B) + static_cast<int64_t>(ok[j] ? wrow : 0) * p.ldb;
  }
  float acc[RPW][MX];  // MX = the activation rows this instance handles (registers)
#pragma unroll
  for (int j = 0; j < RPW; ++j)
#pragma unroll
    for (int m = 0; m < MX; ++m) acc[j][m] = 0.f;
  const __nv_bfloat16* A = reinterpret_cast<const __nv_bfloat16*>(p.A);
#pragma unroll GEMV_UNROLL
  for (int k = lane * 8 + ks * 256; k < K; k += 256 * GEMV_KSPLIT) {
    uint4 wv[RPW];
#pragma unroll
    for (int j = 0; j < RPW; ++j) wv[j] = __ldcs(reinterpret_cast<const uint4*>(w[j] + k));  // streamed once
#pragma unroll
    for (int m = 0; m < MX; ++m) {
      if (m < M) {
        const uint4 av = __ldg(reinterpret_cast<const uint4*>(A + static_cast<int64_t>(m) * p.lda + k));  // L1-resident
        const uint32_t aa[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
        for (int j = 0; j < RPW; ++j) {
          const uint32_t ww[4] = {wv[j].x, wv[j].y, wv[j].z, wv[j].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 a2 = dev::unpack_bf16x2(aa[e]), w2 = dev::unpack_bf16x2(ww[e]);
            acc[j][m] = fmaf(a2.x, w2.x, fmaf(a2.y, w2.y, acc[j][m]));
          }
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < RPW; ++j) {
#pragma unroll
    for (int m = 0; m < MX; ++m) {
#pragma unroll
      for (int x = 16; x > 0; x >>= 1) acc[j][m] += __shfl_xor_sync(0xffffffffu, acc[j][m], x);
    }
    if (lane == 0 && ks > 0) {
      const int rr = warp + 8 * j;
      for (int m = 0; m < M; ++m) spart[ks - 1][rr][m] = acc[j][m];
    }
  }
  if constexpr (GEMV_KSPLIT > 1) __syncthreads();
#pragma unroll
  for (int j = 0; j < RPW; ++j) {
    if (lane == 0 && ks == 0) {
      const int rr = warp + 8 * j;
      for (int m = 0; m < M; ++m) {
        float v = acc[j][m];
        for (int q = 1; q < GEMV_KSPLIT; ++q) v += spart[q - 1][rr][m];
        sout[m][rr] = v;
      }
    }
  }
  __syncthreads();
  const int ncols = min(GEMV_COLS, p.N - c0);
  if (threadIdx.x < M) {
    const int row = threadIdx.x;
    if constexpr (kGlu) {
      __nv_bfloat16* hrow = reinterpret_cast<__nv_bfloat16*>(p.C) + static_cast<int64_t>(row) * p.ldc + c0;
      __nv_bfloat16* prow = reinterpret_cast<__nv_bfloat16*>(p.C2) + static_cast<int64_t>(row) * p.ldc2 + c0;
      for (int c = 0; c < ncols; ++c) {
        const float g = __bfloat162float(__float2bfloat16(sout[row][c]));
        const float u = __bfloat162float(__float2bfloat16(sout[row][GEMV_COLS + c]));
        prow[c] = __float2bfloat16(g);
        prow[p.swiglu_half + c] = __float2bfloat16(u);
        hrow[c] = __float2bfloat16(dev::silu(g) * u);
      }
    } else {
      uint32_t r[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) r[c] = __float_as_uint(c < GEMV_COLS ? sout[row][c] : 0.f);
      epilogue_chunk<EPI>(p, row, c0, ncols, r);
    }
  }
}

// Small-M path on the tensor cores (M <= 8, K % 32 == 0; SwiGLU: gate and up tiles side by side): out^T [16 rows x 8] = W [16 x K] .
// A^T [K x 8] with mma.sync m16n8k16 (bf16 in, fp32 accumulate), the activations as the
// 8-column B operand (columns >= M zero). Each lane streams 16 bytes of two weight rows (g, g+8)
// and 16 bytes of activation row g per 32-deep k step; the contraction order inside a step is
// permuted identically for both operands (lane t's 8 consecutive k feed the fragment slots 2t,
// 2t+1, 2t+8, 2t+9 of two MMAs), so fragments load straight from global memory with 16-byte
// loads. One activation load now serves 16 weight rows (the register kernel re-reads all M
// activation slices from L1 for every pair of rows, which made M = 8 L1-bound at 1.4 TB/s).
// CTA = 16 output columns, 8 warps interleaved along K; partial tiles reduced through shared
// memory, then the common epilogue.
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// NB: 8-row activation groups per warp (the weight fragments of a k step feed NB mmas);
// gridDim.x: groups of 8 * NB activation rows, adjacent CTAs, so the re-reads of a weight tile
// by the CTAs of the other groups hit L2 (M up to GEMV_MMA_MAX_M).
#ifndef SW_GEMV_U
#define SW_GEMV_U 4
#endif
// UX: 32-deep k steps per warp in flight (4; 8 for matrices larger than L2, measured: OPT-66B
// decode 23.3 -> 22.9 ms/token, while the LLaMA-7B-width matrices prefer 4)
template <Epi EPI, int NB, int UX = SW_GEMV_U>
__global__ void __launch_bounds__(256) gemv_mma_kernel(const GemmParams p) {
  constexpr bool kGlu = EPI == Epi::kSwiGLU;  // SwiGLU: gate rows c0.. and up rows swiglu_half + c0..
  constexpr int NT = kGlu ? 2 : 1;
  constexpr int MR = 8 * NB;  // activation rows per CTA
  __shared__ float sred[NT][8][16][MR];
  __shared__ float sout[MR][2 * GEMV_COLS];
  const int K = p.K;
  const int m0 = blockIdx.x * MR;
  const int M = min(MR, p.M - m0);
  const int c0 = blockIdx.y * 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int r_lo = min(c0 + g, p.N - 1), r_hi = min(c0 + g + 8, p.N - 1);
  const __nv_bfloat16* wb = reinterpret_cast<const __nv_bfloat16*>(p.B);
  const __nv_bfloat16* wlo_p[NT];
  const __nv_bfloat16* whi_p[NT];
#pragma unroll
  for (int q = 0; q < NT; ++q) {
    const int off = q ? p.swiglu_half : 0;
    wlo_p[q] = wb + static_cast<int64_t>(off + r_lo) * p.ldb + 8 * t;
    whi_p[q] = wb + static_cast<int64_t>(off + r_hi) * p.ldb + 8 * t;
  }
  const __nv_bfloat16* a_p[NB];
  bool act_row[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    act_row[j] = 8 * j + g < M;
    a_p[j] = reinterpret_cast<const __nv_bfloat16*>(p.A) + static_cast<int64_t>(m0 + (act_row[j] ? 8 * j + g : 0)) * p.lda + 8 * t;
  }
  float acc[NT][NB][4];
#pragma unroll
  for (int q = 0; q < NT; ++q)
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[q][j][0] = acc[q][j][1] = acc[q][j][2] = acc[q][j][3] = 0.f;
  // 32-deep k steps per warp with their loads in flight together
  constexpr int U = NB >= 4 ? 2 : kGlu ? (UX >= 4 ? UX / 2 : 2) : UX;
  // programmatic dependent launch (decode): the weights do not depend on the previous kernel, so
  // the first steps' lines are requested into L2 before waiting for it (a no-op without PDL)
  if (p.pdl) {
    // prefetch depth: measured faster for weight matrices that fit L2 (LLaMA-7B width, 2.64 ->
    // 2.56 ms/token), slower for larger ones (OPT-66B width), where only the early launch is kept
    const bool fits_l2 = static_cast<int64_t>(p.N) * p.K * 2 * NT <= (128ll << 20);
    const int pf_steps = (p.pdl >= 3 && fits_l2) ? 2 * U : (p.pdl == 2 ? U : 0);
#pragma unroll
    for (int u = 0; u < 2 * U; ++u) {
      const int kk = warp * 32 + u * 256;
      if (kk < K && u < pf_steps) {
#pragma unroll
        for (int q = 0; q < NT; ++q) {
          dev::prefetch_l2(wlo_p[q] + kk);
          dev::prefetch_l2(whi_p[q] + kk);
        }
      }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  for (int k = warp * 32; k < K; k += 256 * U) {
    uint4 wl[U][NT], wh[U][NT], av[U][NB];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = k + u * 256;
      if (kk < K) {
#pragma unroll
        for (int q = 0; q < NT; ++q) {
          wl[u][q] = __ldcs(reinterpret_cast<const uint4*>(wlo_p[q] + kk));
          wh[u][q] = __ldcs(reinterpret_cast<const uint4*>(whi_p[q] + kk));
        }
#pragma unroll
        for (int j = 0; j < NB; ++j)
          av[u][j] = act_row[j] ? __ldg(reinterpret_cast<const uint4*>(a_p[j] + kk)) : make_uint4(0, 0, 0, 0);
      } else {
#pragma unroll
        for (int q = 0; q < NT; ++q) wl[u][q] = wh[u][q] = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int j = 0; j < NB; ++j) av[u][j] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int q = 0; q < NT; ++q) {
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          mma_bf16_16816(acc[q][j], wl[u][q].x, wh[u][q].x, wl[u][q].y, wh[u][q].y, av[u][j].x, av[u][j].y);
          mma_bf16_16816(acc[q][j], wl[u][q].z, wh[u][q].z, wl[u][q].w, wh[u][q].w, av[u][j].z, av[u][j].w);
        }
      }
    }
  }
  if (p.pdl) asm volatile("griddepcontrol.launch_dependents;");
  // d0, d1: (row g, activation rows 8j + 2t, 8j + 2t + 1); d2, d3: (row g + 8, same)
#pragma unroll
  for (int q = 0; q < NT; ++q) {
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      sred[q][warp][g][8 * j + 2 * t] = acc[q][j][0];
      sred[q][warp][g][8 * j + 2 * t + 1] = acc[q][j][1];
      sred[q][warp][g + 8][8 * j + 2 * t] = acc[q][j][2];
      sred[q][warp][g + 8][8 * j + 2 * t + 1] = acc[q][j][3];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 16 * M; i += 256) {
    const int r = i & 15, m = i >> 4;
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) v += sred[q][w][r][m];
      sout[m][q * GEMV_COLS + r] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < M) {
    const int lrow = threadIdx.x, row = m0 + lrow;
    const int ncols = min(16, p.N - c0);
    if constexpr (kGlu) {  // the register kernel's SwiGLU epilogue: h = silu(g) * u, pre = g | u (bf16)
      __nv_bfloat16* hrow = reinterpret_cast<__nv_bfloat16*>(p.C) + static_cast<int64_t>(row) * p.ldc + c0;
      __nv_bfloat16* prow = reinterpret_cast<__nv_bfloat16*>(p.C2) + static_cast<int64_t>(row) * p.ldc2 + c0;
      for (int c = 0; c < ncols; ++c) {
        const float gv = __bfloat162float(__float2bfloat16(sout[lrow][c]));
        const float uv = __bfloat162float(__float2bfloat16(sout[lrow][GEMV_COLS + c]));
        prow[c] = __float2bfloat16(gv);
        prow[p.swiglu_half + c] = __float2bfloat16(uv);
        hrow[c] = __float2bfloat16(dev::silu(gv) * uv);
      }
    } else {
      uint32_t rr[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) rr[c] = __float_as_uint(c < 16 ? sout[lrow][c] : 0.f);
      epilogue_chunk<EPI>(p, row, c0, ncols, rr);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Decode-size GEMMs on tcgen05 (9 <= M <= 128 activation rows): swap-AB, C^T[N, M] = W[N, K] .
// A[M, K]^T, so the weight rows fill the 128-lane MMA M dimension and the few activation rows
// are the MMA N (MP = M rounded up to 16; the mma.sync kernel above tops out near 90 TF/s, which
// caps it from M ~ 24 on). One CTA per (128 weight rows, K slice): a TMA ring streams [128 x 64]
// weight boxes, one pass over the weights for the whole job, against [MP x 64] activation boxes
// (L2-resident). The S K-slices of a row block form one thread-block cluster: their fp32
// partials are summed in rank order through distributed shared memory (deterministic, no global
// workspace or counters, graph- and stream-safe), then the rank-0 CTA runs the epilogue shared
// with the other GEMM kernels. Two CTAs per SM (~100 KB of shared memory each).
// ---------------------------------------------------------------------------------------------
template <Epi EPI, int MP>
struct Gtc {
  static constexpr int NT = EPI == Epi::kSwiGLU ? 2 : 1;  // SwiGLU: gate and up tiles
  static constexpr int W_BYTES = 128 * 64 * 2;
  static constexpr int A_BYTES = MP * 64 * 2;
  static constexpr int STAGE = NT * W_BYTES + A_BYTES;
  static constexpr int RAW = (100 * 1024) / STAGE;
  static constexpr int STAGES = RAW < 3 ? 3 : (RAW > 8 ? 8 : RAW);
  static constexpr int ROWP = 129;  // padded row (floats) of the transposed accumulator
  static constexpr int RED = NT * MP * ROWP * 4;
  static constexpr int BODY = STAGES * STAGE > RED ? STAGES * STAGE : RED;
  static constexpr int SMEM = BODY + 256 + 1024;  // + barriers + alignment slack
  static constexpr uint32_t TCOLS = NT * MP <= 32 ? 32 : NT * MP <= 64 ? 64 : NT * MP <= 128 ? 128 : 256;
};

template <Epi EPI, int MP>
__global__ void __launch_bounds__(128, 1) gemv_tc_kernel(const __grid_constant__ CUtensorMap tw,
                                                         const __grid_constant__ CUtensorMap ta, const GemmParams p,
                                                         int S) {
  using G = Gtc<EPI, MP>;
  extern __shared__ uint8_t gtc_raw[];
  uint8_t* sm = gtc_raw + ((1024 - (dev::smem_u32(gtc_raw) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + G::BODY);
  uint64_t* empty = full + G::STAGES;
  uint64_t* done = empty + G::STAGES;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int rb = blockIdx.x / S, s = blockIdx.x - rb * S;  // the cluster: the S slices of row block rb
  const int n0 = rb * 128;
  const int nkb = (p.K + 63) / 64;
  const int kb0 = s * nkb / S, kb1 = (s + 1) * nkb / S;
  if (tid == 0) {
    dev::tma_prefetch_desc(&tw);
    dev::tma_prefetch_desc(&ta);
    for (int i = 0; i < G::STAGES; ++i) {
      dev::mbar_init(&full[i], 1);
      dev::mbar_init(&empty[i], 1);
    }
    dev::mbar_init(done, 1);
    dev::fence_barrier_init();
  }
  if (warp == 2) dev::tmem_alloc<G::TCOLS>(tslot);
  if (p.pdl) {
    // programmatic dependent launch (decode): the first stages' weight rows are requested into L2
    // before waiting for the kernel that produces the activations
    const int nb = min(kb1 - kb0, G::STAGES);
    for (int i = tid; i < 128 * G::NT * nb * 2; i += 128) {
      const int half = i & 1, kb = kb0 + (i >> 1) / (128 * G::NT), rr = ((i >> 1) % (128 * G::NT));
      const int row = (rr < 128 ? n0 + rr : p.swiglu_half + n0 + rr - 128);
      const int64_t rows_total = G::NT == 2 ? 2LL * p.swiglu_half : p.N;
      if (row < rows_total && kb * 64 + half * 32 < p.K)
        dev::prefetch_l2(reinterpret_cast<const __nv_bfloat16*>(p.B) + static_cast<int64_t>(row) * p.ldb + kb * 64 +
                         half * 32);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp == 0) {
    if (lane == 0) {
      for (int kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
        const int st = i % G::STAGES;
        dev::mbar_wait(&empty[st], ((i / G::STAGES) & 1) ^ 1);
        uint8_t* b = sm + st * G::STAGE;
        dev::mbar_arrive_expect_tx(&full[st], G::STAGE);
        dev::tma_load_2d(b, &tw, &full[st], kb * 64, n0);
        if constexpr (G::NT == 2) dev::tma_load_2d(b + G::W_BYTES, &tw, &full[st], kb * 64, p.swiglu_half + n0);
        dev::tma_load_2d(b + G::NT * G::W_BYTES, &ta, &full[st], kb * 64, 0);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = dev::make_idesc_bf16(128, MP, 0, 0);
    for (int kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
      const int st = i % G::STAGES;
      dev::mbar_wait(&full[st], (i / G::STAGES) & 1);
      dev::tc_fence_after();
      const uint32_t b = dev::smem_u32(sm + st * G::STAGE);
      if (dev::elect_one_sync()) {
        const uint64_t da = dev::make_sdesc_sw128(b + G::NT * G::W_BYTES, 16, 1024);
#pragma unroll
        for (int q = 0; q < G::NT; ++q) {
          const uint64_t dw = dev::make_sdesc_sw128(b + q * G::W_BYTES, 16, 1024);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            dev::umma_f16_ss(tmem + q * MP, dw + kk * 2, da + kk * 2, idesc, (i > 0 || kk > 0) ? 1u : 0u);
        }
        dev::umma_commit(&empty[st]);
      }
      __syncwarp();
    }
    if (dev::elect_one_sync()) dev::umma_commit(done);
    __syncwarp();
  }
  // accumulator (lane = weight row n0 + tid, column = activation row) -> transposed in shared
  // memory (the ring is idle: every MMA, hence every TMA load, has completed)
  dev::mbar_wait(done, 0);
  if (p.pdl) asm volatile("griddepcontrol.launch_dependents;");
  dev::tc_fence_after();
  float* sT = reinterpret_cast<float*>(sm);
  const uint32_t lb = static_cast<uint32_t>(warp * 32) << 16;
#pragma unroll 1
  for (int c = 0; c < G::NT * MP; c += 16) {
    uint32_t r[16];
    dev::tmem_ld_32x32b_x16(tmem + lb + c, r);
    dev::tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 16; ++j) sT[(c + j) * G::ROWP + tid] = __uint_as_float(r[j]);
  }
  dev::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    dev::tc_fence_after();
    dev::tmem_dealloc<G::TCOLS>(tmem);
  }
  const int M = p.M;
  // Activation rows m with m % S == s are summed over the S slices (in rank order: the same bits
  // whichever CTA adds them) and written out by this CTA. Only the owner of a row reads the
  // peers' copies of it, so the sum goes back into the owner's own copy in place.
  if (S > 1) {
    dev::cluster_sync();  // every slice's partial is in its shared memory
    const uint32_t base = dev::smem_u32(sT);
#pragma unroll 1
    for (int m = s; m < M; m += S) {
#pragma unroll
      for (int q = 0; q < G::NT; ++q) {
        const int e = (q * MP + m) * G::ROWP + tid;
        float part[8];
#pragma unroll
        for (int r = 0; r < 8; ++r)
          part[r] = r < S ? (r == s ? sT[e] : dev::ld_shared_cluster_f32(dev::mapa_shared(base + e * 4, r))) : 0.f;
        float v = part[0];
#pragma unroll
        for (int r = 1; r < 8; ++r)
          if (r < S) v += part[r];
        sT[e] = v;
      }
    }
    dev::cluster_sync();  // the peers have read this CTA's partials
  }
  __syncthreads();
  const int mine = S > 1 ? (M - s + S - 1) / S : M;  // rows s, s + S, ...
  for (int it = tid; it < mine * 4; it += 128) {
    const int m = s + (it >> 2) * S, cc = it & 3;
    const int col0 = n0 + cc * 32;
    const int ncols = min(32, p.N - col0);
    if (ncols <= 0) continue;
    const float* row = sT + m * G::ROWP + cc * 32;
    if constexpr (EPI == Epi::kSwiGLU) {  // h = silu(g) * u, pre = g | u (bf16), as the other kernels
      __nv_bfloat16* hrow = reinterpret_cast<__nv_bfloat16*>(p.C) + static_cast<int64_t>(m) * p.ldc + col0;
      __nv_bfloat16* prow = reinterpret_cast<__nv_bfloat16*>(p.C2) + static_cast<int64_t>(m) * p.ldc2 + col0;
      for (int c = 0; c < ncols; ++c) {
        const float gv = __bfloat162float(__float2bfloat16(row[c]));
        const float uv = __bfloat162float(__float2bfloat16(row[MP * G::ROWP + c]));
        prow[c] = __float2bfloat16(gv);
        prow[p.swiglu_half + c] = __float2bfloat16(uv);
        hrow[c] = __float2bfloat16(dev::silu(gv) * uv);
      }
    } else {
      uint32_t r[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) r[c] = __float_as_uint(row[c]);
      epilogue_chunk<EPI>(p, m, col0, ncols, r);
    }
  }
}

// SW_GEMV_MMA=0: the register-streamed kernel for every M
bool gemv_mma_on() {
  static const bool on = [] {
    const char* e = std::getenv("SW_GEMV_MMA");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

// Largest M the tensor-core weight-streaming kernel takes (SW_GEMV_MMA_MAX_M); above it the
// tcgen05 GEMM, whose 128-row tiles leave most SMs idle at decode batch sizes (N / 256 CTAs).
int gemv_mma_max_m() {
  static const int v = [] {
    const char* e = std::getenv("SW_GEMV_MMA_MAX_M");
    return e != nullptr ? std::atoi(e) : 64;
  }();
  return v;
}

// Measured on B200 (tools/gemv_bench.py, M = 1): KSPLIT 2 / UNROLL 4 streams N = 4096 weights at
// 2.7-3.9 TB/s (was 2.3-2.6), KSPLIT 1 / UNROLL 2 is best from N = 11008 up (3.1-4.0 TB/s)
template <Epi EPI>
cudaError_t launch_gemv(const GemmParams& p, cudaStream_t stream) {
  {
    static const int mma_min_m = [] {
      // measured: at M = 1 as well the tensor-core kernel streams as fast or faster (4.3-6.1 TB/s)
      const char* e = std::getenv("SW_GEMV_MMA_MIN_M");
      return e != nullptr ? std::atoi(e) : 1;
    }();
    if ((p.M >= mma_min_m || p.M > GEMV_MAX_M) && p.K % 32 == 0 && gemv_mma_on()) {
      const unsigned nt = static_cast<unsigned>((p.N + 15) / 16);
      const bool big = static_cast<int64_t>(p.N) * p.K * 2 * (EPI == Epi::kSwiGLU ? 2 : 1) > (128ll << 20);
      if (p.M <= 8 && p.pdl) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(1, nt);
        cfg.blockDim = dim3(256);
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return big ? cudaLaunchKernelEx(&cfg, gemv_mma_kernel<EPI, 1, 8>, p)
                   : cudaLaunchKernelEx(&cfg, gemv_mma_kernel<EPI, 1>, p);
      } else if (p.M <= 8) {
        if (big) {
          gemv_mma_kernel<EPI, 1, 8><<<dim3(1, nt), 256, 0, stream>>>(p);
        } else {
          gemv_mma_kernel<EPI, 1><<<dim3(1, nt), 256, 0, stream>>>(p);
        }
      } else if (p.M <= 16) {
        gemv_mma_kernel<EPI, 2><<<dim3(1, nt), 256, 0, stream>>>(p);
      } else {
        gemv_mma_kernel<EPI, 4><<<dim3((p.M + 31) / 32, nt), 256, 0, stream>>>(p);
      }
      return cudaGetLastError();
    }
  }
  const int grid = (p.N + GEMV_COLS - 1) / GEMV_COLS;
  // accumulators sized for the actual M: at M = 1 the kernel needs far fewer registers, so more
  // CTAs (and their weight loads) are resident per SM (ncu: 80 registers capped the M <= 8
  // instance at 3 CTAs / 37.5% warps per SM)
  auto go = [&](auto mx) {
    constexpr int MX = decltype(mx)::value;
    if (p.N <= 8192) {
      gemv_bf16_kernel<EPI, 2, 4, MX><<<grid, 512, 0, stream>>>(p);
    } else {
      gemv_bf16_kernel<EPI, 1, 2, MX><<<grid, 256, 0, stream>>>(p);
    }
  };
  if (p.M == 1) {
    go(std::integral_constant<int, 1>{});
  } else if (p.M == 2) {
    go(std::integral_constant<int, 2>{});
  } else if (p.M <= 4) {
    go(std::integral_constant<int, 4>{});
  } else {
    go(std::integral_constant<int, GEMV_MAX_M>{});
  }
  return cudaGetLastError();
}

// SW_GEMV_TC=0: no tcgen05 decode GEMM; SW_GEMV_TC_MIN_M: smallest M it takes (default 9)
bool gemv_tc_on() {
  static const bool on = [] {
    const char* e = std::getenv("SW_GEMV_TC");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

int gemv_tc_min_m() {
  static const int v = [] {
    const char* e = std::getenv("SW_GEMV_TC_MIN_M");
    return e != nullptr ? std::atoi(e) : 9;
  }();
  return v;
}

template <Epi EPI, int MP>
cudaError_t launch_gemv_tc_mp(const GemmParams& p, cudaStream_t stream) {
  using G = Gtc<EPI, MP>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemv_tc_kernel<EPI, MP>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const uint64_t w_rows = EPI == Epi::kSwiGLU ? 2ull * p.swiglu_half : static_cast<uint64_t>(p.N);
  const CUtensorMap tw = make_tmap_bf16_2d(p.B, p.K, w_rows, p.ldb, 64, 128);
  const CUtensorMap ta = make_tmap_bf16_2d(p.A, p.K, p.M, p.lda, 64, MP);
  const int nrb = (p.N + 127) / 128, nkb = (p.K + 63) / 64;
  // K slices per row block: enough CTAs for two per SM, each slice at least two 64-deep blocks
  const int target = 2 * device_sm_count();
  int S = 1;
  while (S < 8 && nrb * S * 2 <= target && nkb / (S * 2) >= 2) S *= 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(nrb * S));
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = G::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = static_cast<unsigned>(S);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = p.pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, gemv_tc_kernel<EPI, MP>, tw, ta, p, S);
}

template <Epi EPI>
cudaError_t launch_gemv_tc(const GemmParams& p, cudaStream_t stream) {
  if (p.M <= 16) return launch_gemv_tc_mp<EPI, 16>(p, stream);
  if (p.M <= 32) return launch_gemv_tc_mp<EPI, 32>(p, stream);
  if (p.M <= 64) return launch_gemv_tc_mp<EPI, 64>(p, stream);
  return launch_gemv_tc_mp<EPI, 128>(p, stream);
}


// The small-M path applies to forward-layout GEMMs whose activations fit in shared memory.
bool gemv_tc_ok(const GemmParams& p) {
  return gemv_tc_on() && p.M >= gemv_tc_min_m() && p.M <= 128 && !p.a_mn_major && !p.b_mn_major && p.K % 8 == 0 &&
         p.lda % 8 == 0 && p.ldb % 8 == 0 &&
         (p.epi == Epi::kStoreBf16 || p.epi == Epi::kStoreF32 || p.epi == Epi::kBiasGelu ||
          p.epi == Epi::kResidF32 || p.epi == Epi::kSwiGLU) &&
         !(p.epi == Epi::kStoreF32 && p.accumulate);
}

bool gemv_ok(const GemmParams& p) {
  return (p.M <= GEMV_MAX_M || (p.M <= gemv_mma_max_m() && p.K % 32 == 0 && gemv_mma_on())) && !p.a_mn_major && !p.b_mn_major && p.K % 8 == 0 && p.lda % 8 == 0 &&
         p.ldb % 8 == 0 &&
         (p.epi == Epi::kStoreBf16 || p.epi == Epi::kStoreF32 || p.epi == Epi::kBiasGelu ||
          p.epi == Epi::kResidF32 || p.epi == Epi::kSwiGLU) &&
         !(p.epi == Epi::kStoreF32 && p.accumulate);
}

}  // namespace

// Split-K for fp32-store weight-gradient GEMMs with too few 256 x 256 tiles for the CTA pairs
// (the shards of tensor-parallel layers: 4096 x 512 at TP = 8 is 32 tiles for 74 pairs): the
// slice count whose units fill the pairs' waves best, with at least 8 k-blocks per slice. At
// most 2 slices by default (SW_GEMM_SPLITK_MAX): two reduce-adds onto the zeroed output commute
// (0 + a + b == 0 + b + a), so the result stays bitwise deterministic; 3+ slices measured only
// 0-2.5% faster on the TP = 8 shapes. Not when accumulating into C (C + a + b would depend on the
// order). SW_GEMM_SPLITK=0 disables; p.split_k > 0 forces.
int choose_split_k(const GemmParams& p) {
  if (p.split_k > 0) return p.split_k;
  static const bool on = [] {
    const char* e = std::getenv("SW_GEMM_SPLITK");
    return !(e != nullptr && e[0] == '0');
  }();
  // weight-gradient layout only (both operands MN-major): the reduce-adds make the sum's order
  // run-dependent, which the activation-gradient path (amplified through the attention
  // backward) should not be
  if (!on || p.accumulate || !p.a_mn_major || !p.b_mn_major || p.bias != nullptr || p.alpha != 1.0f || gemv_ok(p) ||
      gemv_tc_ok(p))
    return 1;
  const int tiles = ((p.M + 2 * BM - 1) / (2 * BM)) * ((p.N + BN - 1) / BN);
  const int pairs = device_sm_count() / 2;
  const int num_kb = (p.K + BK - 1) / BK;
  static const int max_waves = [] {
    const char* e = std::getenv("SW_GEMM_SPLITK_WAVES");
    return e != nullptr ? std::atoi(e) : 2;
  }();
  static const double min_gain = [] {
    const char* e = std::getenv("SW_GEMM_SPLITK_GAIN");
    return e != nullptr ? std::atof(e) : 0.05;
  }();
  static const int max_split = [] {
    const char* e = std::getenv("SW_GEMM_SPLITK_MAX");
    return e != nullptr ? std::max(1, std::min(8, std::atoi(e))) : 2;
  }();
  if (tiles >= max_waves * pairs) return 1;
  int best = 1;
  double best_eff = static_cast<double>(tiles) / (((tiles + pairs - 1) / pairs) * pairs);
  for (int s = 2; s <= max_split && num_kb / s >= 8; ++s) {
    const int units = tiles * s;
    const double eff = static_cast<double>(units) / (((units + pairs - 1) / pairs) * pairs);
    if (eff > best_eff + min_gain) {
      best = s;
      best_eff = eff;
    }
  }
  return best;
}

int gemm_split_k(const GemmParams& p) {
  GemmParams q = p;
  q.epi = Epi::kStoreF32;
  return use_pairs() && SW_EPI_TMA ? choose_split_k(q) : 1;
}

bool gemm_delta_ok(const GemmParams& p) {
  return SW_EPI_TMA && use_pairs() && !p.accumulate && p.aux != nullptr && p.delta != nullptr && p.delta_T > 0 &&
         p.M % p.delta_T == 0 && p.N % 128 == 0 && p.ld_aux % 8 == 0 && p.C2 == nullptr && !gemv_ok(p);
}

bool gemm_colsum_ok(const GemmParams& p) {
  return SW_EPI_TMA && use_pairs() && p.epi == Epi::kGeluBwd && !p.accumulate && !gemv_ok(p);
}

void gemm_trace_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_gemm_trace, sizeof(unsigned long long) * 1024);
}

cudaError_t gemm_bf16(const GemmParams& p, cudaStream_t stream) {
  if (p.M <= 0 || p.N <= 0 || p.K <= 0) {
    throw std::runtime_error("gemm_bf16: empty problem M=" + std::to_string(p.M) +
                             " N=" + std::to_string(p.N) + " K=" + std::to_string(p.K));
  }
  if (p.N % 8 != 0) throw std::runtime_error("gemm_bf16: N must be a multiple of 8");
  if (p.ldc % 8 != 0) throw std::runtime_error("gemm_bf16: ldc must be a multiple of 8");
  if (gemv_tc_ok(p)) {
    switch (p.epi) {
      case Epi::kStoreBf16: return launch_gemv_tc<Epi::kStoreBf16>(p, stream);
      case Epi::kStoreF32: return launch_gemv_tc<Epi::kStoreF32>(p, stream);
      case Epi::kBiasGelu: return launch_gemv_tc<Epi::kBiasGelu>(p, stream);
      case Epi::kResidF32: return launch_gemv_tc<Epi::kResidF32>(p, stream);
      case Epi::kSwiGLU: return launch_gemv_tc<Epi::kSwiGLU>(p, stream);
      default: break;
    }
  }
  if (gemv_ok(p)) {
    switch (p.epi) {
      case Epi::kStoreBf16: return launch_gemv<Epi::kStoreBf16>(p, stream);
      case Epi::kStoreF32: return launch_gemv<Epi::kStoreF32>(p, stream);
      case Epi::kBiasGelu: return launch_gemv<Epi::kBiasGelu>(p, stream);
      case Epi::kResidF32: return launch_gemv<Epi::kResidF32>(p, stream);
      case Epi::kSwiGLU: return launch_gemv<Epi::kSwiGLU>(p, stream);
      default: break;
    }
  }
  if (p.epi == Epi::kStoreF32 && use_pairs() && SW_EPI_TMA) {
    GemmParams q = p;
    q.split_k = choose_split_k(p);
    if (q.split_k > 1) {
      if (!p.accumulate) {
        const cudaError_t e = cudaMemset2DAsync(p.C, static_cast<size_t>(p.ldc) * 4, 0, static_cast<size_t>(p.N) * 4,
                                                static_cast<size_t>(p.M), stream);
        if (e != cudaSuccess) return e;
      }
      return launch<Epi::kStoreF32>(q, stream);
    }
  }
  switch (p.epi) {
    case Epi::kStoreBf16: return launch<Epi::kStoreBf16>(p, stream);
    case Epi::kStoreF32: return launch<Epi::kStoreF32>(p, stream);
    case Epi::kBiasGelu: return launch<Epi::kBiasGelu>(p, stream);
    case Epi::kResidF32: return launch<Epi::kResidF32>(p, stream);
    case Epi::kGeluBwd:
      if (p.colsum != nullptr && !gemm_colsum_ok(p))
        throw std::runtime_error("gemm_bf16: fused column sums not available for this call");
      return launch<Epi::kGeluBwd>(p, stream);
    case Epi::kSwiGLU:
      if (p.swiglu_half != p.N || p.b_mn_major) {
        throw std::runtime_error("gemm_bf16: SwiGLU needs swiglu_half == N and a K-major fused weight");
      }
      return launch<Epi::kSwiGLU>(p, stream);
    case Epi::kSwiGLUBwd:
      if (p.swiglu_half != p.N || p.aux == nullptr) {
        throw std::runtime_error("gemm_bf16: SwiGLU backward needs swiglu_half == N and the pre-activations");
      }
      return launch<Epi::kSwiGLUBwd>(p, stream);
    case Epi::kBf16Delta:
      if (!gemm_delta_ok(p)) throw std::runtime_error("gemm_bf16: fused attention delta not available for this call");
      return launch<Epi::kBf16Delta>(p, stream);
    case Epi::kAdamW: {
      GemmParams q = p;
      const float lo = 1.0f / 16384.0f;
      q.adam_fast = (p.adam_c1 >= lo && p.adam_c1 <= 1.0f && p.adam_c2 >= lo && p.adam_c2 <= 1.0f) ? 1 : 0;
      return launch<Epi::kAdamW>(q, stream);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace sw
