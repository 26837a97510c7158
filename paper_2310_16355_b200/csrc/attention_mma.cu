// tcgen05 flash attention (causal, head-sharded) for head_dim 64 / 128.
//
// Forward, one CTA per (128-query block, batch*head), heaviest (latest) query blocks first:
//   warp 0  TMA producer: Q once, then K_j / V_j into a 2-stage ring (one 2-D tensor map over
//           the fused qkv activations [B*T, 3*Dl], box 64 x 128, SWIZZLE_128B)
//   warp 1  MMA issuer:   S_j = Q K_j^T into one of two TMEM S buffers (128 fp32 columns each);
//           O += P_j V_j into the TMEM O accumulator (P from smem, V as an MN-major operand)
//   warp 2  TMEM allocator (512 columns)
//   warps 4..7 softmax:   thread t owns query row t: reads S_j from TMEM lane t, online softmax
//           with lazy rescaling (O in TMEM is rescaled only when the running max grows by more
//           than 2^8), writes P_j (bf16) into a SWIZZLE_128B smem tile, finally O / l -> bf16.
// S_{j+1} is computed on the tensor core while the softmax warps work on S_j, and P_j V_j
// runs while they work on S_{j+1}.
//
// Backward, one CTA per (128-key block, batch*head) iterating over query blocks i >= j:
//   S^T = K Q_i^T and dP^T = V dO_i^T (TMEM, lane = key), P^T = exp(S^T*scale - lse),
//   dS^T = P^T * (dP^T - delta) * scale written to smem (bf16), then
//   dV += P^T dO_i, dK += dS^T Q_i (TMEM accumulators), dQ_i = dS K (TMEM, lane = query) added
//   to an fp32 dQ accumulator in HBM with vector reductions.
// Every smem tile is a [rows x 64-column] SWIZZLE_128B chunk array, usable both as a K-major
// and as an MN-major UMMA operand, so no tile is ever transposed.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "kernels.h"
#include "sm100.cuh"
#include "tensormap.h"

namespace sw {
namespace k {

namespace {

#ifndef SW_EXP_POLY
#define SW_EXP_POLY 0  // forward softmax: pairs (of every 8) whose exp2 runs as an FMA polynomial
#endif

constexpr int BQ = 128;
constexpr int BKV = 128;
constexpr int CHUNK = 128 * 128;  // bytes of one [128 rows x 64 bf16] SW128 chunk

// Work order of the causal kernels: (batch*head) in groups of G; inside a group the heaviest
// unit (most key/query blocks) of every head first, so the block scheduler's last wave holds the
// lightest units while the G heads of a group still share their K/V or Q/dO reads through L2.
// G <= 0: head-major order (unit fastest). Returns the unit rank (0 = heaviest) and bh.
__device__ __forceinline__ void work_item(int idx, int nunits, int nbh, int G, int& unit, int& bh) {
  if (G <= 0) {
    unit = idx % nunits;
    bh = idx / nunits;
    return;
  }
  const int grp = idx / (G * nunits);
  const int r = idx - grp * G * nunits;
  const int g = min(G, nbh - grp * G);
  unit = r / g;
  bh = grp * G + r % g;
}

// Phase tracing of one CTA (tools/attn_trace.py): clock64 stamps at the pipeline's waits.
__device__ unsigned long long g_attn_trace[4096];
#define ATTN_TR(slot)                                                                \
  do {                                                                               \
    if (static_cast<int>(blockIdx.x) == trace_cta) g_attn_trace[(slot)] = clock64(); \
  } while (0)

int trace_cta() {
  static const int c = [] {
    const char* e = std::getenv("SW_ATTN_TRACE_CTA");
    return e != nullptr ? std::atoi(e) : -1;
  }();
  return c;
}

// SW_ATTN_BWD_TS=0 selects shared-memory P^T / dS^T operands for dV / dK (A/B comparisons).
int bwd_ts() {
  static const int v = [] {
    const char* e = std::getenv("SW_ATTN_BWD_TS");
    return e != nullptr ? std::atoi(e) : 1;
  }();
  return v;
}

// SW_ATTN_DQ_EXT=0: dQ accumulated inside the key-block kernel (dQ^T = K^T dS^T per block, fp32
// TMA reduce-adds into HBM) instead of the dS^T tiles written out for the query-block dQ kernel
int bwd_dq_ext() {
  static const int v = [] {
    const char* e = std::getenv("SW_ATTN_DQ_EXT");
    return e != nullptr ? std::atoi(e) : 1;
  }();
  return v;
}

// dS^T tiles of the causal backward for the dQ kernel: per (batch*head), key block kb holds the
// 64-query chunks n = 0 .. (T - 128 kb) / 64 - 1 (queries 128 kb + 64 n ..), each a [128 keys x
// 64 queries] bf16 SW128 image (16 KiB, the shared-memory layout the MMA reads). Chunk index:
__host__ __device__ __forceinline__ int64_t ds_chunks_before(int kb, int T) {
  return static_cast<int64_t>(kb) * (T / 64) - static_cast<int64_t>(kb) * (kb - 1);
}
__host__ __device__ __forceinline__ int64_t ds_chunk(int bh, int kb, int n, int T) {
  return static_cast<int64_t>(bh) * ds_chunks_before(T / 128, T) + ds_chunks_before(kb, T) + n;
}

int bwd_dq_first() {
  static const int v = [] {
    const char* e = std::getenv("SW_ATTN_BWD_DQ_FIRST");
    return e != nullptr ? std::atoi(e) : 1;
  }();
  return v;
}

int work_group() {
  static const int g = [] {
    const char* e = std::getenv("SW_ATTN_GROUP");
    return e != nullptr ? std::atoi(e) : 8;
  }();
  return g;
}

__device__ __forceinline__ uint64_t kdesc(uint32_t base, int kk) {
  // K-major operand, 16-element K step kk: chunk kk/4, +32 B inside the swizzle row.
  return dev::make_sdesc_sw128(base + (kk >> 2) * CHUNK + (kk & 3) * 32, 16, 1024);
}

__device__ __forceinline__ uint64_t mndesc(uint32_t base, int kk) {
  // MN-major operand whose K runs along the 128 rows of each chunk: 16 rows per step;
  // 64-wide M/N chunks CHUNK bytes apart.
  return dev::make_sdesc_sw128(base + kk * 2048, CHUNK, 1024);
}

template <int HD>
struct FwdLayout {
  static constexpr int Q = BQ * HD * 2;
  static constexpr int KV = BKV * HD * 2;
  static constexpr int P = BQ * BKV * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q;
  static constexpr int OFF_V = OFF_K + 2 * KV;
  static constexpr int OFF_P = OFF_V + 2 * KV;
  static constexpr int OFF_X = OFF_P + 2 * P;  // row max / row sum exchange, [2][2][128] floats
  static constexpr int OFF_BAR = OFF_X + 4 * 128 * 4;
  static constexpr int BYTES = OFF_BAR + 128;  // the dynamic smem base is 1024-aligned (declared)
};

template <int HD>
__global__ void __launch_bounds__(384, 1)
    attn_fwd_tc(const __grid_constant__ CUtensorMap tm, bf16* __restrict__ out, float* __restrict__ lse,
                int T, int Hl, float scale_log2, float scale) {
  using Lay = FwdLayout<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  uint8_t* sQ = smem + Lay::OFF_Q;
  uint8_t* sK = smem + Lay::OFF_K;
  uint8_t* sV = smem + Lay::OFF_V;
  uint8_t* sP = smem + Lay::OFF_P;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;    // [2]
  uint64_t* p_full = bars + 7;    // [2]
  uint64_t* pv_done = bars + 9;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int nqb = (T + BQ - 1) / BQ;
  // consecutive CTAs share (batch, head) so its K/V stays L2-resident; heaviest block first
  const int qb = nqb - 1 - static_cast<int>(blockIdx.x) % nqb;
  const int bh = static_cast<int>(blockIdx.x) / nqb;
  const int b = bh / Hl, h = bh % Hl;
  const int Dl = Hl * HD;
  const int q0 = qb * BQ;
  const int row0 = b * T;
  const int nkv = qb + 1;

  const uint32_t warp = dev::warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&tm);
    dev::mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      dev::mbar_init(&kv_full[i], 1);
      dev::mbar_init(&kv_empty[i], 1);
      dev::mbar_init(&s_full[i], 1);
      dev::mbar_init(&p_full[i], 256);
      dev::mbar_init(&pv_done[i], 1);
    }
    dev::fence_barrier_init();
  }
  if (warp == 2) dev::tmem_alloc<512>(tmem_slot);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_o = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      dev::mbar_arrive_expect_tx(q_full, Lay::Q);
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) dev::tma_load_2d(sQ + c * CHUNK, &tm, q_full, h * HD + c * 64, row0 + q0);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        dev::mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        dev::mbar_arrive_expect_tx(&kv_full[st], 2 * Lay::KV);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          dev::tma_load_2d(sK + st * Lay::KV + c * CHUNK, &tm, &kv_full[st], Dl + h * HD + c * 64, row0 + j * BKV);
          dev::tma_load_2d(sV + st * Lay::KV + c * CHUNK, &tm, &kv_full[st], 2 * Dl + h * HD + c * 64, row0 + j * BKV);
        }
      }
    }
  } else if (warp == 1) {
    // the whole warp runs the issue loop (uniform descriptors); one elected lane issues
    {
      const uint32_t id_s = dev::make_idesc_bf16(BQ, BKV, 0, 0);
      const uint32_t id_o = dev::make_idesc_bf16(BQ, HD, 0, 1);
      const uint64_t dq = dev::make_sdesc_sw128(dev::smem_u32(sQ), 16, 1024);
      const uint64_t dk = dev::make_sdesc_sw128(dev::smem_u32(sK), 16, 1024);
      const uint64_t dp = dev::make_sdesc_sw128(dev::smem_u32(sP), 16, 1024);
      const uint64_t dv = dev::make_sdesc_sw128(dev::smem_u32(sV), CHUNK, 1024);
      auto kstep = [](int kk) { return static_cast<uint64_t>((kk >> 2) * (CHUNK >> 4) + (kk & 3) * 2); };
      dev::mbar_wait(q_full, 0);
      auto issue_pv = [&](int j) {
        const int bb = j & 1;
        dev::mbar_wait(&p_full[bb], (j >> 1) & 1);
        dev::tc_fence_after();
        const uint64_t ap = dp + static_cast<uint64_t>(bb * (Lay::P >> 4));
        const uint64_t bv = dv + static_cast<uint64_t>(bb * (Lay::KV >> 4));
        if (dev::elect_one_sync()) {
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk)
            dev::umma_f16_ss(t_o, ap + kstep(kk), bv + static_cast<uint64_t>(kk * 128), id_o,
                             (j > 0 || kk > 0) ? 1u : 0u);
          dev::umma_commit(&pv_done[bb]);
          dev::umma_commit(&kv_empty[bb]);
        }
        __syncwarp();
      };
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        dev::mbar_wait(&kv_full[st], (j >> 1) & 1);
        dev::tc_fence_after();
        const uint64_t bk = dk + static_cast<uint64_t>(st * (Lay::KV >> 4));
        if (dev::elect_one_sync()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            dev::umma_f16_ss(tmem + st * 128, dq + kstep(kk), bk + kstep(kk), id_s, kk > 0 ? 1u : 0u);
          dev::umma_commit(&s_full[st]);
        }
        __syncwarp();
        if (j >= 1) issue_pv(j - 1);
      }
      issue_pv(nkv - 1);
    }
  } else if (warp >= 4) {
    // Two softmax warpgroups: warps 4-7 own keys [0, 64) of every query row, warps 8-11 keys
    // [64, 128); the row max and the final row sum are exchanged through shared memory.
    const int wg = (static_cast<int>(warp) - 4) >> 2;
    const int r = static_cast<int>(threadIdx.x) - 128 - wg * 128;  // query row within the block
    const int q = q0 + r;
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    float* xm = reinterpret_cast<float*>(smem + Lay::OFF_X);  // [parity][wg][128]
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < nkv; ++j) {
      const int bb = j & 1;
      dev::mbar_wait(&s_full[bb], (j >> 1) & 1);
      dev::tc_fence_after();
      const uint32_t ts = tmem + lane_base + bb * 128 + wg * 64;
      const bool diag = (j == nkv - 1);
      const int key0 = j * BKV + wg * 64;
      uint32_t v[64];
      dev::tmem_ld_32x32b_x32(ts, *reinterpret_cast<uint32_t(*)[32]>(v));
      dev::tmem_ld_32x32b_x32(ts + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
      dev::tmem_ld_wait();
      if (diag) {
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          const int key = key0 + i;
          if (!(key <= q && key < T)) v[i] = __float_as_uint(-INFINITY);
        }
      }
      float mloc = __uint_as_float(v[0]);
#pragma unroll
      for (int i = 1; i < 64; ++i) mloc = fmaxf(mloc, __uint_as_float(v[i]));
      xm[(bb * 2 + wg) * 128 + r] = mloc;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const float mx = fmaxf(mloc, xm[(bb * 2 + (wg ^ 1)) * 128 + r]);
      // lazy rescale: keep the stale max unless the new one is 2^8 larger in exp2 units
      bool resc = false;
      float factor = 1.f;
      if (j == 0) {
        m_used = mx;
      } else if ((mx - m_used) * scale_log2 > 8.f) {
        resc = true;
        factor = dev::ex2_approx((m_used - mx) * scale_log2);
        m_used = mx;
        l *= factor;
      }
      if (__any_sync(0xffffffffu, resc)) {
        // O is rewritten in TMEM: wait for every earlier P V product to land
        dev::mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
        dev::tc_fence_after();
#pragma unroll 1
        for (int c = wg * (HD / 64); c < (wg + 1) * (HD / 64); ++c) {
          uint32_t o[32];
          dev::tmem_ld_32x32b_x32(t_o + lane_base + c * 32, o);
          dev::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * factor);
          dev::tmem_st_32x32b_x32(t_o + lane_base + c * 32, o);
        }
        dev::tmem_st_wait();
      }
      // the P buffer bb was last read by P_{j-2} V_{j-2}
      if (j >= 2) dev::mbar_wait(&pv_done[bb], ((j - 2) >> 1) & 1);
      const float mb = m_used * scale_log2;
      uint8_t* tile = sP + bb * Lay::P;
      float ls = 0.f;
#pragma unroll
      for (int c = 0; c < 8; ++c) {  // 8 units of 8 keys
        uint32_t pk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float p0 = dev::ex2_approx(fmaf(__uint_as_float(v[8 * c + 2 * e]), scale_log2, -mb));
          const float p1 = dev::ex2_approx(fmaf(__uint_as_float(v[8 * c + 2 * e + 1]), scale_log2, -mb));
          ls += p0 + p1;
          pk[e] = dev::pack_bf16x2(p0, p1);
        }
        dev::st_sw128(tile, BQ, r, wg, c, make_uint4(pk[0], pk[1], pk[2], pk[3]));
      }
      l += ls;
      dev::fence_proxy_async_smem();
      dev::tc_fence_before();
      dev::mbar_arrive(&p_full[bb]);
    }
    // epilogue: O / l with l summed over both halves (the other parity's exchange slots were
    // last read before the final block's barrier)
    const int xp = ((nkv - 1) & 1) ^ 1;
    xm[(xp * 2 + wg) * 128 + r] = l;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    l += xm[(xp * 2 + (wg ^ 1)) * 128 + r];
    dev::mbar_wait(&pv_done[(nkv - 1) & 1], ((nkv - 1) >> 1) & 1);
    dev::tc_fence_after();
    const float inv = 1.f / l;
    bf16* orow = out + (static_cast<int64_t>(row0) + q) * Dl + h * HD;
#pragma unroll
    for (int c = wg * (HD / 64); c < (wg + 1) * (HD / 64); ++c) {
      uint32_t v[32];
      dev::tmem_ld_32x32b_x32(t_o + lane_base + c * 32, v);
      dev::tmem_ld_wait();
      if (q < T) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint4 w;
          w.x = dev::pack_bf16x2(__uint_as_float(v[8 * u + 0]) * inv, __uint_as_float(v[8 * u + 1]) * inv);
          w.y = dev::pack_bf16x2(__uint_as_float(v[8 * u + 2]) * inv, __uint_as_float(v[8 * u + 3]) * inv);
          w.z = dev::pack_bf16x2(__uint_as_float(v[8 * u + 4]) * inv, __uint_as_float(v[8 * u + 5]) * inv);
          w.w = dev::pack_bf16x2(__uint_as_float(v[8 * u + 6]) * inv, __uint_as_float(v[8 * u + 7]) * inv);
          *reinterpret_cast<uint4*>(orow + c * 32 + 8 * u) = w;
        }
      }
    }
    if (wg == 0 && q < T) lse[static_cast<int64_t>(bh) * T + q] = m_used * scale + logf(l);
  }
  dev::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    dev::tc_fence_after();
    dev::tmem_dealloc<512>(tmem);
  }
}

template <int HD>
bool launch_fwd(const bf16* qkv, bf16* o, float* lse, int B, int T, int Hl, cudaStream_t s) {
  using Lay = FwdLayout<HD>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(attn_fwd_tc<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay::BYTES) !=
        cudaSuccess) {
      return false;
    }
    configured = true;
  }
  const int Dl = Hl * HD;
  const CUtensorMap tm = make_tmap_bf16_2d(qkv, 3ull * Dl, static_cast<uint64_t>(B) * T, 3ull * Dl, 64, 128);
  const int nqb = (T + BQ - 1) / BQ;
  const double scale = 1.0 / std::sqrt(static_cast<double>(HD));
  attn_fwd_tc<HD><<<nqb * B * Hl, 384, Lay::BYTES, s>>>(tm, o, lse, T, Hl,
                                                         static_cast<float>(scale * 1.4426950408889634),
                                                         static_cast<float>(scale));
  return true;
}


// ---------------------------------------------------------------------------------------------
// forward, two query tiles per CTA (head_dim 128): each softmax warpgroup owns a whole 128-row
// query tile (lane = row, all 128 keys of a block: no cross-warpgroup max exchange), and the two
// tiles ping-pong on the tensor core -- while one warpgroup turns S into P, the MMA warp runs
// the other tile's S = Q K^T and O += P V. P goes back into the S columns of TMEM as bf16 and
// feeds the O MMA straight from TMEM (tcgen05.mma with A in tensor memory).
//   TMEM: S_A | O_A | S_B | O_B (128 columns each)
//   smem: Q_A, Q_B, and a 2-stage K/V ring shared by both tiles
// ---------------------------------------------------------------------------------------------
struct Fwd2Layout {
  static constexpr int HD = 128;
  static constexpr int Q = 128 * HD * 2;
  static constexpr int KV = 128 * HD * 2;
  static constexpr int OFF_QA = 0;
  static constexpr int OFF_QB = OFF_QA + Q;
  static constexpr int OFF_K = OFF_QB + Q;       // [2]
  static constexpr int OFF_V = OFF_K + 2 * KV;   // [2]
  static constexpr int OFF_BAR = OFF_V + 2 * KV;
  static constexpr int BYTES = OFF_BAR + 256;
};

// Item order of the persistent kernels: the work list (heaviest first, work_item) is dealt to
// the P resident CTAs in snake order (round r: CTA c takes position c, or P-1-c on odd rounds),
// so each CTA's summed work stays close to the mean without a dynamic scheduler.
__device__ __forceinline__ int snake_item(int round, int c, int P) {
  return round * P + ((round & 1) ? P - 1 - c : c);
}

// Persistent: a CTA walks its items (snake_item) and keeps the pipeline full across them -- the
// K/V ring runs on without a break, the next item's Q_t is loaded as soon as tile t's last
// S = Q K^T has executed (q_empty), and a softmax warpgroup writes its O while the tensor core
// already runs the next item's first S. Barrier phases count blocks / items per CTA, not per
// item. With gridDim.x == the item count every CTA takes one item (the non-persistent launch).
__global__ void __launch_bounds__(384, 1)
    attn_fwd_tc2(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm_kv,
                 bf16* __restrict__ out, float* __restrict__ lse, int T, int Tk, int kcol, int vcol, int Hl,
                 float scale_log2, float scale, int nbh, int group, int causal, const float* __restrict__ lut,
                 int trace_cta) {
  // T queries per sequence from tm (q at column h*HD); Tk keys from tm_kv (k at kcol + h*HD,
  // v at vcol + h*HD). Self-attention: tm_kv == tm, Tk == T, kcol = Dl, vcol = 2 Dl (fused
  // q|k|v); cross-attention (T5): separate encoder K/V, Tk != T allowed (non-causal, no bias).
  using Lay = Fwd2Layout;
  constexpr int HD = Lay::HD;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ[2] = {smem + Lay::OFF_QA, smem + Lay::OFF_QB};
  uint8_t* sK = smem + Lay::OFF_K;
  uint8_t* sV = smem + Lay::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::OFF_BAR);
  uint64_t* q_full = bars + 0;    // [tile]
  uint64_t* q_empty = bars + 2;   // [tile] the tile's last S of the item has executed
  uint64_t* kv_full = bars + 4;   // [2]
  uint64_t* kv_empty = bars + 6;  // [2]
  uint64_t* s_full = bars + 8;    // [tile]
  uint64_t* p_full = bars + 10;   // [tile]
  uint64_t* pv_done = bars + 12;  // [tile]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

  const int nqb = (T + 127) / 128;
  const int npair = (nqb + 1) / 2;
  const int nitems = npair * nbh;
  const int Dl = Hl * HD;
  // additive relative-position bias (T5): lut[h][key - query + T - 1] in natural units, row
  // pitch 2T + 128; the scores are then scale * s + bias and the exp2 runs in log2(e) units
  const float sl_eff = lut ? 1.4426950408889634f : scale_log2;
  const float sc_eff = lut ? 1.f : scale;
  // the item's geometry: pair index, (batch, head), and the key blocks of each query tile
  struct Item {
    int bh, h, row0, row0k, qa, nkv, nkv_t[2];
    bool hasB;
  };
  auto item_of = [&](int idx) {
    Item it;
    int rank_;
    work_item(idx, npair, nbh, group, rank_, it.bh);
    const int pi = npair - 1 - rank_;  // heaviest pair first
    it.h = it.bh % Hl;
    it.row0 = (it.bh / Hl) * T;
    it.row0k = (it.bh / Hl) * Tk;
    it.qa = 2 * pi;
    it.hasB = it.qa + 1 < nqb;
    // causal: key blocks up to the diagonal; otherwise (T5 encoder / cross) every key block
    const int nkb = (Tk + 127) / 128;
    it.nkv_t[0] = causal ? it.qa + 1 : nkb;
    it.nkv_t[1] = it.hasB ? (causal ? it.qa + 2 : nkb) : 0;
    it.nkv = causal ? (it.hasB ? it.qa + 2 : it.qa + 1) : nkb;
    return it;
  };
  const int P = static_cast<int>(gridDim.x), cta = static_cast<int>(blockIdx.x);

  const uint32_t warp = dev::warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&tm);
    dev::tma_prefetch_desc(&tm_kv);
    for (int i = 0; i < 2; ++i) {
      dev::mbar_init(&q_full[i], 1);
      dev::mbar_init(&q_empty[i], 1);
      dev::mbar_init(&kv_full[i], 1);
      dev::mbar_init(&kv_empty[i], 1);
      dev::mbar_init(&s_full[i], 1);
      dev::mbar_init(&p_full[i], 128);
      dev::mbar_init(&pv_done[i], 1);
    }
    dev::fence_barrier_init();
  }
  if (warp == 2) dev::tmem_alloc<512>(tmem_slot);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0 && static_cast<int>(blockIdx.x) == trace_cta) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    g_attn_trace[4090] = clock64();
    g_attn_trace[4091] = gt;
  }

  if (warp == 0) {
    if (lane == 0) {
      int gj = 0;               // K/V blocks loaded so far (ring slot gj & 1)
      int cq[2] = {0, 0};       // items loaded per query tile
      for (int r = 0;; ++r) {
        const int idx = snake_item(r, cta, P);
        if (idx >= nitems) break;
        const Item it = item_of(idx);
        for (int t = 0; t < (it.hasB ? 2 : 1); ++t) {
          if (cq[t] > 0) dev::mbar_wait(&q_empty[t], (cq[t] - 1) & 1);
          dev::mbar_arrive_expect_tx(&q_full[t], Lay::Q);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c)
            dev::tma_load_2d(sQ[t] + c * CHUNK, &tm, &q_full[t], it.h * HD + c * 64, it.row0 + (it.qa + t) * 128);
          ++cq[t];
        }
        for (int j = 0; j < it.nkv; ++j, ++gj) {
          const int st = gj & 1;
          dev::mbar_wait(&kv_empty[st], ((gj >> 1) & 1) ^ 1);
          dev::mbar_arrive_expect_tx(&kv_full[st], 2 * Lay::KV);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c) {
            dev::tma_load_2d(sK + st * Lay::KV + c * CHUNK, &tm_kv, &kv_full[st], kcol + it.h * HD + c * 64,
                             it.row0k + j * 128);
            dev::tma_load_2d(sV + st * Lay::KV + c * CHUNK, &tm_kv, &kv_full[st], vcol + it.h * HD + c * 64,
                             it.row0k + j * 128);
          }
        }
      }
    }
  } else if (warp == 1) {
    // whole warp runs the schedule; one elected lane issues
    const uint32_t id_s = dev::make_idesc_bf16(128, 128, 0, 0);
    const uint32_t id_o = dev::make_idesc_bf16(128, HD, 0, 1);
    const uint64_t dq[2] = {dev::make_sdesc_sw128(dev::smem_u32(sQ[0]), 16, 1024),
                            dev::make_sdesc_sw128(dev::smem_u32(sQ[1]), 16, 1024)};
    const uint64_t dk = dev::make_sdesc_sw128(dev::smem_u32(sK), 16, 1024);
    const uint64_t dv = dev::make_sdesc_sw128(dev::smem_u32(sV), CHUNK, 1024);
    auto kstep = [](int kk) { return static_cast<uint64_t>((kk >> 2) * (CHUNK >> 4) + (kk & 3) * 2); };
    int gj = 0;              // K/V blocks consumed before this item
    int ct[2] = {0, 0};      // blocks of each tile before this item (s_full / p_full / pv_done phases)
    int cq[2] = {0, 0};
    for (int r = 0;; ++r) {
      const int idx = snake_item(r, cta, P);
      if (idx >= nitems) break;
      const Item it = item_of(idx);
      // S_t(j) = Q_t K_j^T; after the tile's last block, Q_t may be replaced (q_empty)
      auto issue_s = [&](int t, int j) {
        const uint64_t bk = dk + static_cast<uint64_t>(((gj + j) & 1) * (Lay::KV >> 4));
        if (dev::elect_one_sync()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            dev::umma_f16_ss(tmem + t * 256, dq[t] + kstep(kk), bk + kstep(kk), id_s, kk > 0 ? 1u : 0u);
          dev::umma_commit(&s_full[t]);
          if (j == it.nkv_t[t] - 1) dev::umma_commit(&q_empty[t]);
        }
        __syncwarp();
      };
      auto issue_pv = [&](int t, int j) {
        const int tb = (ct[t] + j) * 16 + 2 * t;  // trace: blocks of this CTA, per tile
        if (lane == 0 && tb < 3900) ATTN_TR(tb);
        dev::mbar_wait(&p_full[t], (ct[t] + j) & 1);
        if (lane == 0 && tb < 3900) ATTN_TR(tb + 1);
        dev::tc_fence_after();
        const uint64_t bv = dv + static_cast<uint64_t>(((gj + j) & 1) * (Lay::KV >> 4));
        if (dev::elect_one_sync()) {
#pragma unroll
          for (int kk = 0; kk < 128 / 16; ++kk)  // P (bf16 pairs) sits in the first 64 columns of S
            dev::umma_f16_ts(tmem + t * 256 + 128, tmem + t * 256 + kk * 8, bv + static_cast<uint64_t>(kk * 128), id_o,
                             (j > 0 || kk > 0) ? 1u : 0u);
          dev::umma_commit(&pv_done[t]);
        }
        __syncwarp();
      };
      if (lane == 0 && cq[0] < 16) ATTN_TR(4000 + 4 * cq[0]);
      dev::mbar_wait(&q_full[0], cq[0] & 1);
      if (it.hasB) dev::mbar_wait(&q_full[1], cq[1] & 1);
      if (lane == 0 && cq[0] < 16) ATTN_TR(4001 + 4 * cq[0]);
      dev::mbar_wait(&kv_full[gj & 1], (gj >> 1) & 1);
      if (lane == 0 && cq[0] < 16) ATTN_TR(4002 + 4 * cq[0]);
      dev::tc_fence_after();
      issue_s(0, 0);
      if (it.hasB) issue_s(1, 0);
      for (int j = 0; j < it.nkv; ++j) {
        if (j < it.nkv_t[0]) issue_pv(0, j);
        if (j + 1 < it.nkv) {
          dev::mbar_wait(&kv_full[(gj + j + 1) & 1], ((gj + j + 1) >> 1) & 1);
          dev::tc_fence_after();
        }
        if (j + 1 < it.nkv_t[0]) issue_s(0, j + 1);
        if (j < it.nkv_t[1]) issue_pv(1, j);
        if (j + 1 < it.nkv_t[1]) issue_s(1, j + 1);
        if (dev::elect_one_sync()) dev::umma_commit(&kv_empty[(gj + j) & 1]);  // K_j / V_j consumed
        __syncwarp();
      }
      gj += it.nkv;
      ct[0] += it.nkv_t[0];
      ct[1] += it.nkv_t[1];
      ++cq[0];
      if (it.hasB) ++cq[1];
    }
  } else if (warp >= 4) {
    const int t = (static_cast<int>(warp) - 4) >> 2;  // query tile of this warpgroup
    const int r = static_cast<int>(warp & 3) * 32 + static_cast<int>(lane);
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_base + t * 256, tO = tS + 128;
    int ct = 0;  // this tile's blocks before the item
    for (int rr = 0;; ++rr) {
      const int idx = snake_item(rr, cta, P);
      if (idx >= nitems) break;
      const Item it = item_of(idx);
      if (t == 1 && !it.hasB) continue;
      const int h = it.h, bh = it.bh;
      const int q = (it.qa + t) * 128 + r;
      const int nk = it.nkv_t[t];
      float m_used = -INFINITY, l = 0.f;
      const bool trw = lane == 0 && (warp & 3) == 0;
      for (int j = 0; j < nk; ++j) {
        const int tb = (ct + j) * 16 + 4 + 4 * t;
        if (trw && tb < 3900) ATTN_TR(tb);
        dev::mbar_wait(&s_full[t], (ct + j) & 1);
        if (trw && tb < 3900) ATTN_TR(tb + 1);
        dev::tc_fence_after();
        uint32_t v[128];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          dev::tmem_ld_32x32b_x32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * c));
        dev::tmem_ld_wait();
        auto bias_mask = [&]() {
          if (lut) {
            const float* lr = lut + static_cast<int64_t>(h) * (2 * T + 128) + (T - 1 - (q < T ? q : T - 1)) + j * 128;
#pragma unroll
            for (int i = 0; i < 128; ++i) v[i] = __float_as_uint(fmaf(__uint_as_float(v[i]), scale, __ldg(lr + i)));
          }
          if ((causal && j == nk - 1) || (j + 1) * 128 > Tk) {
#pragma unroll
            for (int i = 0; i < 128; ++i) {
              const int key = j * 128 + i;
              if (!((!causal || key <= q) && key < Tk)) v[i] = __float_as_uint(-INFINITY);
            }
          }
        };
        bias_mask();
        // Lazy rescale (FA4-style): the running max m_used moves only when a row's block max
        // exceeds it by more than 2^8 in exp2 units. After block 0 the exps are taken against
        // m_used straight away while the block max is reduced alongside them (independent
        // chains, no max -> exp dependency on the critical path); a row whose max did jump
        // takes the rare slow path: O is rescaled and P is recomputed from S, still in TMEM.
        // The O rewrite uses warp-collective TMEM loads/stores, so the whole warp takes it
        // together (factor 1 for the rows that keep their max).
        const float2 sl2 = make_float2(sl_eff, sl_eff);
        float l_blk;
        auto exps = [&](float mref) {  // P in place: v[e] = bf16x2(p[2e], p[2e+1]); returns the row sum
          const float mb = mref * sl_eff;
          const float2 nmb2 = make_float2(-mb, -mb);
          float2 ls[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
          for (int e = 0; e < 64; ++e) {
            const float2 a = dev::ffma2(make_float2(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1])), sl2, nmb2);
            // SW_EXP_POLY of every 8 pairs on the FMA pipe, the rest on MUFU
            const float2 pp = (e & 7) < SW_EXP_POLY ? dev::ex2_poly2(a)
                                                    : make_float2(dev::ex2_approx(a.x), dev::ex2_approx(a.y));
            ls[e & 3] = dev::fadd2(ls[e & 3], pp);
            v[e] = dev::pack_bf16x2(pp.x, pp.y);
          }
          const float2 s01 = dev::fadd2(ls[0], ls[1]), s23 = dev::fadd2(ls[2], ls[3]);
          return (s01.x + s23.x) + (s01.y + s23.y);
        };
        auto rowmax = [&]() {
          float m4[4] = {__uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]), __uint_as_float(v[3])};
#pragma unroll
          for (int i = 4; i < 128; i += 8) {
#pragma unroll
            for (int u = 0; u < 4; ++u) m4[u] = dev::fmax3(m4[u], __uint_as_float(v[i + 2 * u]), __uint_as_float(v[i + 2 * u + 1]));
          }
          return fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
        };
        if (j == 0) {
          m_used = rowmax();
          l_blk = exps(m_used);
        } else {
          // block max from the raw scores before exps() overwrites them (the reductions and the
          // exps are independent, so the scheduler interleaves them)
          const float mx = rowmax();
          l_blk = exps(m_used);
          const bool resc = (mx - m_used) * sl_eff > 8.f;
          if (__any_sync(0xffffffffu, resc)) {
            const float factor = resc ? dev::ex2_approx((m_used - mx) * sl_eff) : 1.f;
            if (resc) {
              m_used = mx;
              l *= factor;
            }
            dev::mbar_wait(&pv_done[t], (ct + j - 1) & 1);  // every earlier P V has landed in O
            dev::tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < HD / 32; ++c) {
              uint32_t o[32];
              dev::tmem_ld_32x32b_x32(tO + c * 32, o);
              dev::tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * factor);
              dev::tmem_st_32x32b_x32(tO + c * 32, o);
            }
            dev::tmem_st_wait();
            // P again against the new max: S_j is still in TMEM (reload, re-bias, re-mask)
#pragma unroll
            for (int c = 0; c < 4; ++c)
              dev::tmem_ld_32x32b_x32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * c));
            dev::tmem_ld_wait();
            bias_mask();
            l_blk = exps(m_used);
          }
        }
        dev::tmem_st_32x32b_x32(tS, *reinterpret_cast<uint32_t(*)[32]>(v));
        dev::tmem_st_32x32b_x32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        l += l_blk;
        if (trw && tb < 3900) ATTN_TR(tb + 2);
        dev::tmem_st_wait();
        dev::tc_fence_before();
        dev::mbar_arrive(&p_full[t]);
        if (trw && tb < 3900) ATTN_TR(tb + 3);
      }
      // O of this item; the next item's first P V (which overwrites O) waits for this warpgroup's
      // next p_full, so the TMEM reads below are done before it
      dev::mbar_wait(&pv_done[t], (ct + nk - 1) & 1);
      dev::tc_fence_after();
      const float inv = 1.f / l;
      bf16* orow = out + (static_cast<int64_t>(it.row0) + q) * Dl + h * HD;
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t o[32];
        dev::tmem_ld_32x32b_x32(tO + c * 32, o);
        dev::tmem_ld_wait();
        if (q < T) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint4 w;
            w.x = dev::pack_bf16x2(__uint_as_float(o[8 * u + 0]) * inv, __uint_as_float(o[8 * u + 1]) * inv);
            w.y = dev::pack_bf16x2(__uint_as_float(o[8 * u + 2]) * inv, __uint_as_float(o[8 * u + 3]) * inv);
            w.z = dev::pack_bf16x2(__uint_as_float(o[8 * u + 4]) * inv, __uint_as_float(o[8 * u + 5]) * inv);
            w.w = dev::pack_bf16x2(__uint_as_float(o[8 * u + 6]) * inv, __uint_as_float(o[8 * u + 7]) * inv);
            *reinterpret_cast<uint4*>(orow + c * 32 + 8 * u) = w;
          }
        }
      }
      if (q < T) lse[static_cast<int64_t>(bh) * T + q] = m_used * sc_eff + logf(l);
      if (trw && t == 0 && rr < 16) ATTN_TR(4003 + 4 * rr);
      dev::tc_fence_before();
      ct += nk;
    }
  }
  dev::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0 && static_cast<int>(blockIdx.x) == trace_cta) {
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    g_attn_trace[4092] = clock64();
    g_attn_trace[4093] = gt;
  }
  if (warp == 2) {
    dev::tc_fence_after();
    dev::tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------------------------------------
// forward v3 (head_dim 128, causal self-attention): two query tiles per CTA as in v2, but 64-key
// blocks with each tile's S double-buffered, so a tile's S_{j+1} = Q K_{j+1}^T executes while its
// softmax warpgroup works on S_j (v2's single S buffer per tile serialised softmax -> P V -> S
// per tile). TMEM per tile: O (128 columns) | S0 (64) | S1 (64); P_j (bf16) over S_j's first 32.
//   warp 0  TMA: Q_A, Q_B once; K_j / V_j ([64 keys x 128] each) into a 4-stage ring
//   warp 1  MMA: per key block j: S_A(j), S_B(j), then P_A(j-1) V_{j-1}, P_B(j-1) V_{j-1}
//   warps 4-7 / 8-11  softmax of tile A / B (thread = query row), lazy running max
// ---------------------------------------------------------------------------------------------
constexpr int F3_BK = 64;
constexpr int F3_NST = 4;
constexpr int F3_CH = F3_BK * 128;  // [64 rows x 64 bf16] SW128 chunk: 8 KiB
struct Fwd3Layout {
  static constexpr int HD = 128;
  static constexpr int Q = 128 * HD * 2;     // 32 KiB
  static constexpr int KV = F3_BK * HD * 2;  // 16 KiB
  static constexpr int OFF_QA = 0;
  static constexpr int OFF_QB = OFF_QA + Q;
  static constexpr int OFF_K = OFF_QB + Q;           // [F3_NST]
  static constexpr int OFF_V = OFF_K + F3_NST * KV;  // [F3_NST]
  static constexpr int OFF_BAR = OFF_V + F3_NST * KV;
  static constexpr int BYTES = OFF_BAR + 256;
};

__global__ void __launch_bounds__(384, 1)
    attn_fwd_tc3(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv,
                 bf16* __restrict__ out, float* __restrict__ lse, int T, int Hl, float scale_log2, float scale,
                 int nbh, int group) {
  using Lay = Fwd3Layout;
  constexpr int HD = Lay::HD;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ[2] = {smem + Lay::OFF_QA, smem + Lay::OFF_QB};
  uint8_t* sK = smem + Lay::OFF_K;
  uint8_t* sV = smem + Lay::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::OFF_BAR);
  uint64_t* q_full = bars;                   // 1
  uint64_t* kv_full = bars + 1;              // [F3_NST]
  uint64_t* kv_empty = kv_full + F3_NST;     // [F3_NST]
  uint64_t* s_full = kv_empty + F3_NST;      // [tile][2]
  uint64_t* p_full = s_full + 4;             // [tile][2]
  uint64_t* pv_done = p_full + 4;            // [tile][2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 4);

  const int nqb = (T + 127) / 128;
  const int npair = (nqb + 1) / 2;
  int rank_, bh;
  work_item(static_cast<int>(blockIdx.x), npair, nbh, group, rank_, bh);
  const int pi = npair - 1 - rank_;  // heaviest pair first
  const int h = bh % Hl;
  const int row0 = (bh / Hl) * T;
  const int qa = 2 * pi;
  const bool hasB = qa + 1 < nqb;
  const int nkt = (T + F3_BK - 1) / F3_BK;
  // causal: 64-key blocks through each tile's diagonal
  const int nk_t[2] = {min(2 * (qa + 1), nkt), hasB ? min(2 * (qa + 2), nkt) : 0};
  const int nkv = hasB ? nk_t[1] : nk_t[0];
  const int Dl = Hl * HD;

  const uint32_t warp = dev::warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&tm_q);
    dev::tma_prefetch_desc(&tm_kv);
    dev::mbar_init(q_full, 1);
    for (int i = 0; i < F3_NST; ++i) {
      dev::mbar_init(&kv_full[i], 1);
      dev::mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      dev::mbar_init(&s_full[i], 1);
      dev::mbar_init(&p_full[i], 128);
      dev::mbar_init(&pv_done[i], 1);
    }
    dev::fence_barrier_init();
  }
  if (warp == 2) dev::tmem_alloc<512>(tmem_slot);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      dev::mbar_arrive_expect_tx(q_full, Lay::Q * (hasB ? 2 : 1));
      for (int t = 0; t < (hasB ? 2 : 1); ++t) {
#pragma unroll
        for (int c = 0; c < HD / 64; ++c)
          dev::tma_load_2d(sQ[t] + c * CHUNK, &tm_q, q_full, h * HD + c * 64, row0 + (qa + t) * 128);
      }
      for (int j = 0; j < nkv; ++j) {
        const int st = j % F3_NST;
        dev::mbar_wait(&kv_empty[st], ((j / F3_NST) & 1) ^ 1);
        dev::mbar_arrive_expect_tx(&kv_full[st], 2 * Lay::KV);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          dev::tma_load_2d(sK + st * Lay::KV + c * F3_CH, &tm_kv, &kv_full[st], Dl + h * HD + c * 64, row0 + j * F3_BK);
          dev::tma_load_2d(sV + st * Lay::KV + c * F3_CH, &tm_kv, &kv_full[st], 2 * Dl + h * HD + c * 64,
                           row0 + j * F3_BK);
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t id_s = dev::make_idesc_bf16(128, F3_BK, 0, 0);
    const uint32_t id_o = dev::make_idesc_bf16(128, HD, 0, 1);
    const uint64_t dq[2] = {dev::make_sdesc_sw128(dev::smem_u32(sQ[0]), 16, 1024),
                            dev::make_sdesc_sw128(dev::smem_u32(sQ[1]), 16, 1024)};
    const uint64_t dk = dev::make_sdesc_sw128(dev::smem_u32(sK), 16, 1024);
    const uint64_t dv = dev::make_sdesc_sw128(dev::smem_u32(sV), F3_CH, 1024);
    constexpr uint64_t KV16 = Lay::KV >> 4;
    auto kq = [](int kk) { return static_cast<uint64_t>((kk >> 2) * (CHUNK >> 4) + (kk & 3) * 2); };   // Q: 128-row chunks
    auto kk64 = [](int kk) { return static_cast<uint64_t>((kk >> 2) * (F3_CH >> 4) + (kk & 3) * 2); }; // K: 64-row chunks
    auto tS = [&](int t, int j) { return tmem + t * 256 + 128 + (j & 1) * 64; };
    auto issue_pv = [&](int t, int j) {
      dev::mbar_wait(&p_full[2 * t + (j & 1)], (j >> 1) & 1);
      dev::tc_fence_after();
      const uint64_t bv = dv + (j % F3_NST) * KV16;
      if (dev::elect_one_sync()) {
#pragma unroll
        for (int kk = 0; kk < F3_BK / 16; ++kk)  // P (bf16 pairs) in the first 32 columns of S_t(j)
          dev::umma_f16_ts(tmem + t * 256, tS(t, j) + kk * 8, bv + static_cast<uint64_t>(kk * 128), id_o,
                           (j > 0 || kk > 0) ? 1u : 0u);
        dev::umma_commit(&pv_done[2 * t + (j & 1)]);
      }
      __syncwarp();
    };
    dev::mbar_wait(q_full, 0);
    for (int j = 0; j < nkv; ++j) {
      const int st = j % F3_NST;
      dev::mbar_wait(&kv_full[st], (j / F3_NST) & 1);
      dev::tc_fence_after();
      const uint64_t bk = dk + st * KV16;
      if (dev::elect_one_sync()) {
        // S_t(j) goes into the buffer of P_t(j-2), whose P V was issued (and so executes) before it
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          if (j < nk_t[t]) {
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk)
              dev::umma_f16_ss(tS(t, j), dq[t] + kq(kk), bk + kk64(kk), id_s, kk > 0 ? 1u : 0u);
            dev::umma_commit(&s_full[2 * t + (j & 1)]);
          }
        }
      }
      __syncwarp();
      if (j >= 1) {
        if (j - 1 < nk_t[0]) issue_pv(0, j - 1);
        if (j - 1 < nk_t[1]) issue_pv(1, j - 1);
        if (dev::elect_one_sync()) dev::umma_commit(&kv_empty[(j - 1) % F3_NST]);  // K/V_{j-1} consumed
        __syncwarp();
      }
    }
    if (nk_t[0] == nkv) issue_pv(0, nkv - 1);
    if (nk_t[1] == nkv) issue_pv(1, nkv - 1);
    if (dev::elect_one_sync()) dev::umma_commit(&kv_empty[(nkv - 1) % F3_NST]);
    __syncwarp();
  } else if (warp >= 4) {
    const int t = (static_cast<int>(warp) - 4) >> 2;
    if (t == 0 || hasB) {
      const int r = static_cast<int>(warp & 3) * 32 + static_cast<int>(lane);
      const int q = (qa + t) * 128 + r;
      const int nk = nk_t[t];
      const uint32_t lb = static_cast<uint32_t>((warp & 3) * 32) << 16;
      const uint32_t tO = tmem + lb + t * 256;
      const float2 sl2 = make_float2(scale_log2, scale_log2);
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < nk; ++j) {
        dev::mbar_wait(&s_full[2 * t + (j & 1)], (j >> 1) & 1);
        dev::tc_fence_after();
        const uint32_t tSj = tmem + lb + t * 256 + 128 + (j & 1) * 64;
        uint32_t v[64];
        auto load_s = [&]() {
          dev::tmem_ld_32x32b_x32(tSj, *reinterpret_cast<uint32_t(*)[32]>(v));
          dev::tmem_ld_32x32b_x32(tSj + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
          dev::tmem_ld_wait();
          if ((j + 1) * F3_BK > (qa + t) * 128 || (j + 1) * F3_BK > T) {
#pragma unroll
            for (int i = 0; i < F3_BK; ++i) {
              const int key = j * F3_BK + i;
              if (key > q || key >= T) v[i] = __float_as_uint(-INFINITY);
            }
          }
        };
        auto rowmax = [&]() {
          float m4[4] = {__uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]), __uint_as_float(v[3])};
#pragma unroll
          for (int i = 4; i < F3_BK; i += 8) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              m4[u] = dev::fmax3(m4[u], __uint_as_float(v[i + 2 * u]), __uint_as_float(v[i + 2 * u + 1]));
          }
          return fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
        };
        auto exps = [&](float mref) {  // P in place: v[e] = bf16x2(p[2e], p[2e+1]); returns the row sum
          const float mb = mref * scale_log2;
          const float2 nmb2 = make_float2(-mb, -mb);
          float2 ls[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
          for (int e = 0; e < F3_BK / 2; ++e) {
            const float2 a = dev::ffma2(make_float2(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1])), sl2, nmb2);
            const float2 pp = make_float2(dev::ex2_approx(a.x), dev::ex2_approx(a.y));
            ls[e & 3] = dev::fadd2(ls[e & 3], pp);
            v[e] = dev::pack_bf16x2(pp.x, pp.y);
          }
          const float2 s01 = dev::fadd2(ls[0], ls[1]), s23 = dev::fadd2(ls[2], ls[3]);
          return (s01.x + s23.x) + (s01.y + s23.y);
        };
        load_s();
        float l_blk;
        if (j == 0) {
          m_used = rowmax();
          l_blk = exps(m_used);
        } else {
          const float mx = rowmax();
          l_blk = exps(m_used);
          const bool resc = (mx - m_used) * scale_log2 > 8.f;
          if (__any_sync(0xffffffffu, resc)) {
            const float factor = resc ? dev::ex2_approx((m_used - mx) * scale_log2) : 1.f;
            if (resc) {
              m_used = mx;
              l *= factor;
            }
            dev::mbar_wait(&pv_done[2 * t + ((j - 1) & 1)], ((j - 1) >> 1) & 1);  // every earlier P V is in O
            dev::tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < HD / 32; ++c) {
              uint32_t o[32];
              dev::tmem_ld_32x32b_x32(tO + c * 32, o);
              dev::tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * factor);
              dev::tmem_st_32x32b_x32(tO + c * 32, o);
            }
            dev::tmem_st_wait();
            load_s();  // S_j is still in TMEM: P again against the new max
            l_blk = exps(m_used);
          }
        }
        l += l_blk;
        dev::tmem_st_32x32b_x32(tSj, *reinterpret_cast<uint32_t(*)[32]>(v));
        dev::tmem_st_wait();
        dev::tc_fence_before();
        dev::mbar_arrive(&p_full[2 * t + (j & 1)]);
      }
      dev::mbar_wait(&pv_done[2 * t + ((nk - 1) & 1)], ((nk - 1) >> 1) & 1);
      dev::tc_fence_after();
      const float inv = 1.f / l;
      bf16* orow = out + (static_cast<int64_t>(row0) + q) * Dl + h * HD;
#pragma unroll 1
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t o[32];
        dev::tmem_ld_32x32b_x32(tO + c * 32, o);
        dev::tmem_ld_wait();
        if (q < T) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            uint4 w;
            w.x = dev::pack_bf16x2(__uint_as_float(o[8 * u + 0]) * inv, __uint_as_float(o[8 * u + 1]) * inv);
            w.y = dev::pack_bf16x2(__uint_as_float(o[8 * u + 2]) * inv, __uint_as_float(o[8 * u + 3]) * inv);
            w.z = dev::pack_bf16x2(__uint_as_float(o[8 * u + 4]) * inv, __uint_as_float(o[8 * u + 5]) * inv);
            w.w = dev::pack_bf16x2(__uint_as_float(o[8 * u + 6]) * inv, __uint_as_float(o[8 * u + 7]) * inv);
            *reinterpret_cast<uint4*>(orow + c * 32 + 8 * u) = w;
          }
        }
      }
      if (q < T) lse[static_cast<int64_t>(bh) * T + q] = m_used * scale + logf(l);
    }
  }
  dev::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    dev::tc_fence_after();
    dev::tmem_dealloc<512>(tmem);
  }
}

// SW_ATTN_FWD3=0: the v2 forward (128-key blocks, one S buffer per tile) for causal self-attention
bool fwd3_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SW_ATTN_FWD3");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

bool launch_fwd3(const bf16* qkv, bf16* o, float* lse, int B, int T, int Hl, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(attn_fwd_tc3, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd3Layout::BYTES) !=
        cudaSuccess) {
      return false;
    }
    configured = true;
  }
  constexpr int HD = 128;
  const int Dl = Hl * HD;
  const CUtensorMap tm_q = make_tmap_bf16_2d(qkv, 3ull * Dl, static_cast<uint64_t>(B) * T, 3ull * Dl, 64, 128);
  const CUtensorMap tm_kv = make_tmap_bf16_2d(qkv, 3ull * Dl, static_cast<uint64_t>(B) * T, 3ull * Dl, 64, F3_BK);
  const int nqb = (T + 127) / 128;
  const int npair = (nqb + 1) / 2;
  const double scale = 1.0 / std::sqrt(static_cast<double>(HD));
  attn_fwd_tc3<<<npair * B * Hl, 384, Fwd3Layout::BYTES, s>>>(tm_q, tm_kv, o, lse, T, Hl,
                                                              static_cast<float>(scale * 1.4426950408889634),
                                                              static_cast<float>(scale), B * Hl, work_group());
  return true;
}

// SW_ATTN_PERSIST=1: one resident CTA per SM walking several items (snake order). Measured
// on B200 (tools/attn_bench.py, LLaMA-7B heads): equal at T = 2048 (the next item's Q load and
// the pipeline refill are not hidden by it), 25% slower at T = 8192 (the hardware's in-order
// block dispatch keeps a head group's K/V reads together in L2, the static deal does not), so
// the default launches one CTA per item.
bool attn_persist() {
  static const bool on = [] {
    const char* e = std::getenv("SW_ATTN_PERSIST");
    return e != nullptr && e[0] == '1';
  }();
  return on;
}

bool fwd2_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SW_ATTN_FWD_V1");
    return !(e != nullptr && e[0] == '1');
  }();
  return on;
}

// kv == nullptr: self-attention over the fused q|k|v rows of qkv; otherwise cross-attention: q
// rows [B*T, ldq] (column h*128), k / v rows [B*Tk, ldkv] with k at kv + h*128, v at kv + voff
bool launch_fwd2(const bf16* qkv, bf16* o, float* lse, int B, int T, int Hl, cudaStream_t s, int causal = 1,
                 const float* lut = nullptr, float scale_arg = 0.f, const bf16* kv = nullptr, int Tk = 0,
                 int64_t ldq = 0, int64_t ldkv = 0, int voff = 0) {
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(attn_fwd_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd2Layout::BYTES) !=
        cudaSuccess) {
      return false;
    }
    configured = true;
  }
  constexpr int HD = 128;
  const int Dl = Hl * HD;
  const bool cross = kv != nullptr;
  const uint64_t lq = cross ? static_cast<uint64_t>(ldq) : 3ull * Dl;
  const CUtensorMap tm = make_tmap_bf16_2d(qkv, cross ? static_cast<uint64_t>(Dl) : 3ull * Dl,
                                           static_cast<uint64_t>(B) * T, lq, 64, 128);
  const CUtensorMap tm_kv = cross ? make_tmap_bf16_2d(kv, static_cast<uint64_t>(voff + Dl), static_cast<uint64_t>(B) * Tk,
                                                      static_cast<uint64_t>(ldkv), 64, 128)
                                  : tm;
  const int nqb = (T + 127) / 128;
  const int npair = (nqb + 1) / 2;
  const double scale = scale_arg > 0.f ? scale_arg : 1.0 / std::sqrt(static_cast<double>(HD));
  const int nitems = npair * B * Hl;
  const int grid = attn_persist() ? std::min(nitems, device_sm_count()) : nitems;
  attn_fwd_tc2<<<grid, 384, Fwd2Layout::BYTES, s>>>(tm, tm_kv, o, lse, T, cross ? Tk : T, cross ? 0 : Dl,
                                                    cross ? voff : 2 * Dl, Hl,
                                                              static_cast<float>(scale * 1.4426950408889634),
                                                              static_cast<float>(scale), B * Hl, work_group(), causal,
                                                              lut, trace_cta());
  return true;
}

// ---------------------------------------------------------------------------------------------
// backward
// ---------------------------------------------------------------------------------------------
template <int HD>
struct BwdLayout {
  static constexpr int T_ = 128 * HD * 2;  // one [128 x HD] bf16 tile
  static constexpr int PT = 128 * 128 * 2;
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + T_;
  static constexpr int OFF_Q = OFF_V + T_;
  static constexpr int OFF_DO = OFF_Q + T_;
  static constexpr int OFF_PT = OFF_DO + T_;
  static constexpr int OFF_DST = OFF_PT + PT;
  static constexpr int OFF_STAT = OFF_DST + PT;   // [2][2][128] floats: lse, delta (double buffered)
  static constexpr int OFF_BAR = OFF_STAT + 2 * 2 * 128 * 4;
  static constexpr int BYTES = OFF_BAR + 256 + 1024;
};

template <int HD>
__global__ void __launch_bounds__(384, 1)
    attn_bwd_tc(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                const __grid_constant__ CUtensorMap tm_dq,
                const float* __restrict__ lse, const float* __restrict__ delta, float* __restrict__ dq_acc,
                bf16* __restrict__ dqkv, int T, int Hl, float scale_log2, float scale) {
  using Lay = BwdLayout<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem + Lay::OFF_K;
  uint8_t* sV = smem + Lay::OFF_V;
  uint8_t* sQ = smem + Lay::OFF_Q;
  uint8_t* sDO = smem + Lay::OFF_DO;
  uint8_t* sPt = smem + Lay::OFF_PT;
  uint8_t* sDSt = smem + Lay::OFF_DST;
  float* sStat = reinterpret_cast<float*>(smem + Lay::OFF_STAT);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::OFF_BAR);
  uint64_t* kv_full = bars + 0;
  uint64_t* qdo_full = bars + 1;
  uint64_t* qdo_empty = bars + 2;
  uint64_t* st_full = bars + 3;
  uint64_t* p_full = bars + 4;
  uint64_t* mma_done = bars + 5;
  uint64_t* dq_free = bars + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

  const int nb = (T + 127) / 128;
  // consecutive CTAs share (batch, head) (Q/dO stay L2-resident); key block 0 has the most work
  const int kb = static_cast<int>(blockIdx.x) % nb;
  const int bh = static_cast<int>(blockIdx.x) / nb;
  const int b = bh / Hl, h = bh % Hl;
  const int Dl = Hl * HD;
  const int key0 = kb * 128;
  const int row0 = b * T;
  const int nq = nb - kb;  // query blocks kb .. nb-1

  const uint32_t warp = dev::warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&tm_qkv);
    dev::tma_prefetch_desc(&tm_do);
    dev::tma_prefetch_desc(&tm_dq);
    dev::mbar_init(kv_full, 1);
    dev::mbar_init(qdo_full, 1);
    dev::mbar_init(qdo_empty, 1);
    dev::mbar_init(st_full, 1);
    dev::mbar_init(p_full, 256);
    dev::mbar_init(mma_done, 1);
    dev::mbar_init(dq_free, 256);
    dev::fence_barrier_init();
  }
  if (warp == 2) dev::tmem_alloc<512>(tmem_slot);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_s = tmem, t_dp = tmem + 128, t_dv = tmem + 256, t_dk = tmem + 256 + HD, t_dq = tmem;

  if (warp == 0) {
    if (lane == 0) {
      dev::mbar_arrive_expect_tx(kv_full, 2 * Lay::T_);
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) {
        dev::tma_load_2d(sK + c * CHUNK, &tm_qkv, kv_full, Dl + h * HD + c * 64, row0 + key0);
        dev::tma_load_2d(sV + c * CHUNK, &tm_qkv, kv_full, 2 * Dl + h * HD + c * 64, row0 + key0);
      }
      for (int n = 0; n < nq; ++n) {
        const int qs = (kb + n) * 128;
        dev::mbar_wait(qdo_empty, (n & 1) ^ 1);
        dev::mbar_arrive_expect_tx(qdo_full, 2 * Lay::T_);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          dev::tma_load_2d(sQ + c * CHUNK, &tm_qkv, qdo_full, h * HD + c * 64, row0 + qs);
          dev::tma_load_2d(sDO + c * CHUNK, &tm_do, qdo_full, h * HD + c * 64, row0 + qs);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_s = dev::make_idesc_bf16(128, 128, 0, 0);
      const uint32_t id_kv = dev::make_idesc_bf16(128, HD, 0, 1);
      const uint32_t id_q = dev::make_idesc_bf16(128, HD, 1, 1);
      const uint32_t aK = dev::smem_u32(sK), aV = dev::smem_u32(sV), aQ = dev::smem_u32(sQ);
      const uint32_t aDO = dev::smem_u32(sDO), aPt = dev::smem_u32(sPt), aDSt = dev::smem_u32(sDSt);
      dev::mbar_wait(kv_full, 0);
      for (int n = 0; n < nq; ++n) {
        dev::mbar_wait(qdo_full, n & 1);
        if (n >= 1) dev::mbar_wait(dq_free, (n - 1) & 1);
        dev::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) dev::umma_f16_ss(t_s, kdesc(aK, kk), kdesc(aQ, kk), id_s, kk > 0);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) dev::umma_f16_ss(t_dp, kdesc(aV, kk), kdesc(aDO, kk), id_s, kk > 0);
        dev::umma_commit(st_full);
        dev::mbar_wait(p_full, n & 1);
        dev::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          dev::umma_f16_ss(t_dv, kdesc(aPt, kk), mndesc(aDO, kk), id_kv, (n > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          dev::umma_f16_ss(t_dk, kdesc(aDSt, kk), mndesc(aQ, kk), id_kv, (n > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) dev::umma_f16_ss(t_dq, mndesc(aDSt, kk), mndesc(aK, kk), id_q, kk > 0);
        dev::umma_commit(mma_done);
        dev::umma_commit(qdo_empty);
      }
    }
  } else if (warp >= 4) {
    // Two softmax warpgroups: warps 4-7 take query columns [0, 64) of every key row, warps 8-11
    // columns [64, 128) (TMEM lane quarter = warp % 4 for both).
    const int wg = (static_cast<int>(warp) - 4) >> 2;                     // 0 or 1
    const int t = static_cast<int>(threadIdx.x) - 128 - wg * 128;        // key row (S^T lane) / query row (dQ lane)
    const int tid = static_cast<int>(threadIdx.x) - 128;                 // 0..255
    const int key = key0 + t;
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const float log2e = 1.4426950408889634f;
    uint8_t* stage = wg == 0 ? sPt : sDSt;  // dQ staging tile of this warpgroup (free after mma_done)
    for (int n = 0; n < nq; ++n) {
      const int qs = (kb + n) * 128;
      float* st_lse = sStat + (n & 1) * 256;
      float* st_del = st_lse + 128;
      if (tid < 128) {
        const int qq = qs + tid;
        st_lse[tid] = qq < T ? lse[static_cast<int64_t>(bh) * T + qq] * log2e : 0.f;
      } else {
        const int qq = qs + tid - 128;
        st_del[tid - 128] = qq < T ? delta[static_cast<int64_t>(bh) * T + qq] : 0.f;
      }
      if (t == 0) dev::bulk_wait_read();  // sPt / sDSt double as the dQ staging tiles
      asm volatile("bar.sync 1, 256;" ::: "memory");
      dev::mbar_wait(st_full, n & 1);
      dev::tc_fence_after();
      if (n >= 1) dev::mbar_wait(mma_done, (n - 1) & 1);  // sPt / sDSt free again
      const bool diag = (n == 0);
      {
        const int half = wg;
        // 64 query columns of S^T and dP^T: four TMEM loads in flight, one wait
        uint32_t sv[64], pv[64];
        dev::tmem_ld_32x32b_x32(t_s + lane_base + half * 64, *reinterpret_cast<uint32_t(*)[32]>(sv));
        dev::tmem_ld_32x32b_x32(t_s + lane_base + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
        dev::tmem_ld_32x32b_x32(t_dp + lane_base + half * 64, *reinterpret_cast<uint32_t(*)[32]>(pv));
        dev::tmem_ld_32x32b_x32(t_dp + lane_base + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(pv + 32));
        dev::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 8; ++u) {  // 8 units of 8 query columns
          uint32_t pk[4], dk[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float pp[2], dd[2];
#pragma unroll
            for (int w2 = 0; w2 < 2; ++w2) {
              const int ci = 8 * u + 2 * e + w2;  // column within the half
              const int qi = half * 64 + ci;
              const int qq = qs + qi;
              float p = dev::ex2_approx(fmaf(__uint_as_float(sv[ci]), scale_log2, -st_lse[qi]));
              const bool ok = qq < T && key < T && (!diag || qq >= key);
              p = ok ? p : 0.f;
              pp[w2] = p;
              dd[w2] = p * (__uint_as_float(pv[ci]) - st_del[qi]) * scale;
            }
            pk[e] = dev::pack_bf16x2(pp[0], pp[1]);
            dk[e] = dev::pack_bf16x2(dd[0], dd[1]);
          }
          dev::st_sw128(sPt, 128, t, half, u, make_uint4(pk[0], pk[1], pk[2], pk[3]));
          dev::st_sw128(sDSt, 128, t, half, u, make_uint4(dk[0], dk[1], dk[2], dk[3]));
        }
      }
      dev::fence_proxy_async_smem();
      dev::tc_fence_before();
      dev::mbar_arrive(p_full);
      // dQ_i rows (TMEM lane = query row): each warpgroup stages HD/2 fp32 columns in SW128
      // tiles (32 columns each) and TMA reduce-adds them into the fp32 dQ accumulator
      // (rows past T carry zeros: dS is masked there).
      dev::mbar_wait(mma_done, n & 1);
      dev::tc_fence_after();
      constexpr int HALF = HD / 2;
      uint32_t v[HALF];
#pragma unroll
      for (int c = 0; c < HALF / 32; ++c)
        dev::tmem_ld_32x32b_x32(t_dq + lane_base + wg * HALF + c * 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * c));
      dev::tmem_ld_wait();
      dev::tc_fence_before();
      dev::mbar_arrive(dq_free);  // TMEM read: the next S^T may overwrite it
#pragma unroll
      for (int bx = 0; bx < HALF / 32; ++bx) {
        uint8_t* tile = stage + bx * 16384;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = bx * 32 + u * 4;
          *reinterpret_cast<uint4*>(tile + t * 128 + ((u ^ (t & 7)) << 4)) = make_uint4(v[c], v[c + 1], v[c + 2], v[c + 3]);
        }
      }
      dev::fence_proxy_async_smem();
      if (wg == 0) {
        asm volatile("bar.sync 2, 128;" ::: "memory");
      } else {
        asm volatile("bar.sync 3, 128;" ::: "memory");
      }
      if (t == 0) {
#pragma unroll
        for (int bx = 0; bx < HALF / 32; ++bx)
          dev::tma_reduce_add_2d(&tm_dq, stage + bx * 16384, h * HD + wg * HALF + bx * 32, row0 + qs);
        dev::bulk_commit();
      }
    }
    if (t == 0) dev::bulk_wait_all();
    // dK, dV (lane = key row) -> bf16 rows of dqkv; each warpgroup writes HD/2 columns
    dev::mbar_wait(mma_done, (nq - 1) & 1);
    dev::tc_fence_after();
    const int64_t ld = 3LL * Dl;
    bf16* dk_row = dqkv + (static_cast<int64_t>(row0) + key) * ld + Dl + h * HD;
    bf16* dv_row = dk_row + Dl;
#pragma unroll 1
    for (int c = wg * (HD / 64); c < (wg + 1) * (HD / 64); ++c) {
      uint32_t a[32], v[32];
      dev::tmem_ld_32x32b_x32(t_dk + lane_base + c * 32, a);
      dev::tmem_ld_32x32b_x32(t_dv + lane_base + c * 32, v);
      dev::tmem_ld_wait();
      if (key < T) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint4 w, z;
          w.x = dev::pack_bf16x2(__uint_as_float(a[8 * u + 0]), __uint_as_float(a[8 * u + 1]));
          w.y = dev::pack_bf16x2(__uint_as_float(a[8 * u + 2]), __uint_as_float(a[8 * u + 3]));
          w.z = dev::pack_bf16x2(__uint_as_float(a[8 * u + 4]), __uint_as_float(a[8 * u + 5]));
          w.w = dev::pack_bf16x2(__uint_as_float(a[8 * u + 6]), __uint_as_float(a[8 * u + 7]));
          z.x = dev::pack_bf16x2(__uint_as_float(v[8 * u + 0]), __uint_as_float(v[8 * u + 1]));
          z.y = dev::pack_bf16x2(__uint_as_float(v[8 * u + 2]), __uint_as_float(v[8 * u + 3]));
          z.z = dev::pack_bf16x2(__uint_as_float(v[8 * u + 4]), __uint_as_float(v[8 * u + 5]));
          z.w = dev::pack_bf16x2(__uint_as_float(v[8 * u + 6]), __uint_as_float(v[8 * u + 7]));
          *reinterpret_cast<uint4*>(dk_row + c * 32 + 8 * u) = w;
          *reinterpret_cast<uint4*>(dv_row + c * 32 + 8 * u) = z;
        }
      }
    }
  }
  dev::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    dev::tc_fence_after();
    dev::tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------------------------------------
// backward, pipelined (head_dim 128): one CTA per (128-key block, batch*head) iterating over
// 64-query blocks. Query-block n+1's S^T / dP^T MMAs run on the tensor core while the softmax
// warpgroups turn block n's S^T / dP^T into P^T / dS^T, and block n's dQ leaves TMEM through a
// separate warpgroup, so the per-block chain no longer serialises the tensor pipe.
//   warp 0      TMA: K, V once; Q_n / dO_n into a 3-deep ring (64-row boxes)
//   warp 1      MMA: S^T_n = K Q_n^T, dP^T_n = V dO_n^T (TMEM, double-buffered, lane = key);
//               then dV += P^T dO_n, dK += dS^T Q_n (TMEM accumulators) and
//               dQ^T_n = K^T dS^T_n (into S^T_n's TMEM columns, lane = head dim)
//   warp 2      TMEM allocator (512 columns: S^T x2 | dP^T x2 | dV | dK)
//   warps 4-11  two softmax warpgroups, 32 query columns each (lane = key row)
//   warps 12-15 dQ warpgroup: dQ^T_n (lane = head dim) -> SW128 fp32 staging -> TMA reduce-add
//               into the fp32 dQ accumulator
// ---------------------------------------------------------------------------------------------
constexpr int BQ2 = 64;
constexpr int CHUNK64 = 64 * 128;  // bytes of one [64 rows x 64 bf16] SW128 chunk

__device__ __forceinline__ uint64_t kdesc64(uint32_t base, int kk) {
  return dev::make_sdesc_sw128(base + (kk >> 2) * CHUNK64 + (kk & 3) * 32, 16, 1024);
}

__device__ __forceinline__ uint64_t mndesc64(uint32_t base, int kk) {
  return dev::make_sdesc_sw128(base + kk * 2048, CHUNK64, 1024);
}

constexpr int QST = 3;  // Q / dO ring depth

struct Bwd2Layout {
  static constexpr int HD = 128;
  static constexpr int KV = 128 * HD * 2;     // 32 KiB
  static constexpr int QT = BQ2 * HD * 2;     // 16 KiB
  static constexpr int PT = 128 * BQ2 * 2;    // 16 KiB: [128 keys x 64 queries] bf16
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + KV;
  static constexpr int OFF_Q = OFF_V + KV;         // [QST]
  static constexpr int OFF_DO = OFF_Q + QST * QT;  // [QST]
  static constexpr int OFF_PT = OFF_DO + QST * QT;
  static constexpr int DQS = BQ2 * HD * 4;    // 32 KiB: dQ staging, 4 boxes of [64 rows x 32 fp32]
  static constexpr int OFF_DST = OFF_PT + PT;
  static constexpr int OFF_DQS = OFF_DST + PT;
  static constexpr int OFF_STAT = OFF_DQS + DQS;  // [2][2][64] floats: lse, delta
  static constexpr int OFF_BAR = OFF_STAT + 2 * 2 * BQ2 * 4;
  static constexpr int BYTES = OFF_BAR + 256;  // dynamic smem base declared 1024-aligned
};

// Column sums across a warp: lane i holds row i of a 32x32 tile in x[]; returns the sum of
// column `lane` (transpose-reduce: 31 shuffles, fixed order).
__device__ __forceinline__ float warp_colsum32(float (&x)[32], uint32_t lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float send = up ? x[i] : x[i + s];
      const float keep = up ? x[i + s] : x[i];
      x[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return x[0];
}

__global__ void __launch_bounds__(512, 1)
    attn_bwd_tc2(const __grid_constant__ CUtensorMap tm_qkv64, const __grid_constant__ CUtensorMap tm_qkv128,
                 const __grid_constant__ CUtensorMap tm_do64, const __grid_constant__ CUtensorMap tm_dq,
                 const float* __restrict__ lse, const float* __restrict__ delta, bf16* __restrict__ dqkv, int T,
                 int Hl, float scale_log2, float scale, int nbh, int group, int trace_cta, int dq_first, int ts,
                 int causal, const float* __restrict__ lut, float* __restrict__ dlut,
                 float* __restrict__ colsum, int Tk, int kcol, int vcol, bf16* __restrict__ dkv, int64_t ld_dkv,
                 int dvoff, uint8_t* __restrict__ ds_out) {
  // ds_out != nullptr (causal self-attention, ts, T % 128 == 0): dQ is not formed here; the dQ
  // warpgroup copies each block's dS^T (bf16, from the dP^T columns of tensor memory) to its
  // ds_chunk() tile for attn_bwd_dq, so the dQ^T MMA, the dS^T shared-memory tile and the fp32
  // dQ staging leave this kernel
  // T queries (tm_qkv64 / tm_do64 / tm_dq rows b*T), Tk keys (tm_qkv128 rows b*Tk, k at kcol,
  // v at vcol); dK / dV rows go to dkv (row pitch ld_dkv, dV at +dvoff). Self-attention: Tk == T,
  // kcol = Dl, vcol = 2 Dl, dkv = dqkv + Dl, ld_dkv = 3 Dl, dvoff = Dl.
  using Lay = Bwd2Layout;
  constexpr int HD = Lay::HD;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sK = smem + Lay::OFF_K;
  uint8_t* sV = smem + Lay::OFF_V;
  uint8_t* sQ = smem + Lay::OFF_Q;
  uint8_t* sDO = smem + Lay::OFF_DO;
  uint8_t* sPt = smem + Lay::OFF_PT;
  uint8_t* sDSt = smem + Lay::OFF_DST;
  uint8_t* sDQ = smem + Lay::OFF_DQS;
  float* sStat = reinterpret_cast<float*>(smem + Lay::OFF_STAT);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::OFF_BAR);
  uint64_t* kv_full = bars + 0;
  uint64_t* qdo_full = bars + 1;   // [QST]
  uint64_t* qdo_empty = bars + 4;  // [QST]
  uint64_t* s_full = bars + 7;     // [2]
  uint64_t* s_free = bars + 9;     // [2]  dQ^T of the block two back has left TMEM
  uint64_t* p_full = bars + 11;
  uint64_t* mma_done = bars + 12;
  uint64_t* dq_full = bars + 13;   // [2]  dQ^T_n is in S^T buffer n & 1
  uint64_t* ds_read = bars + 15;   // the dQ warpgroup has read dS^T_n for the bias gradient
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);
  uint64_t* acc_done = bars + 17;  // every MMA of the CTA complete: dV / dK final

  const int nb = (Tk + 127) / 128;
  int kb, bh;
  work_item(static_cast<int>(blockIdx.x), nb, nbh, group, kb, bh);  // kb 0 = most query blocks
  const int b = bh / Hl, h = bh % Hl;
  const int Dl = Hl * HD;
  const int key0 = kb * 128;
  const int row0 = b * T;
  const int row0k = b * Tk;
  // causal: 64-query blocks from the diagonal on; otherwise (T5 encoder / cross) all of them
  const int qbase = causal ? key0 : 0;
  const int nq = (T - qbase + BQ2 - 1) / BQ2;
  // T5 relative bias: lut / dlut [Hl][2T + 128], index key - query + T - 1 (requires ts: the
  // bias-gradient accumulator takes the otherwise unused P^T tile)
  const float* lut_h = lut ? lut + static_cast<int64_t>(h) * (2 * T + 128) : nullptr;
  float* sAcc = reinterpret_cast<float*>(smem + Lay::OFF_PT);  // [T + 128] when dlut

  const uint32_t warp = dev::warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    ATTN_TR(4000);
    if (static_cast<int>(blockIdx.x) == trace_cta) {
      g_attn_trace[4001] = static_cast<unsigned long long>(nq);
      for (int i = 0; i < 64; ++i) g_attn_trace[i * 16 + 15] = 0;
    }
  }
  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&tm_qkv64);
    dev::tma_prefetch_desc(&tm_qkv128);
    dev::tma_prefetch_desc(&tm_do64);
    dev::tma_prefetch_desc(&tm_dq);
    dev::mbar_init(kv_full, 1);
    for (int i = 0; i < QST; ++i) {
      dev::mbar_init(&qdo_full[i], 1);
      dev::mbar_init(&qdo_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      dev::mbar_init(&s_full[i], 1);
      dev::mbar_init(&s_free[i], 128);
      dev::mbar_init(&dq_full[i], 1);
    }
    dev::mbar_init(p_full, 256);
    dev::mbar_init(ds_read, 128);
    dev::mbar_init(mma_done, 1);
    dev::mbar_init(acc_done, 1);
    dev::fence_barrier_init();
  }
  if (warp == 2) dev::tmem_alloc<512>(tmem_slot);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_s = tmem, t_dp = tmem + 128, t_dv = tmem + 256, t_dk = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      dev::mbar_arrive_expect_tx(kv_full, 2 * Lay::KV);
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) {
        dev::tma_load_2d(sK + c * CHUNK, &tm_qkv128, kv_full, kcol + h * HD + c * 64, row0k + key0);
        dev::tma_load_2d(sV + c * CHUNK, &tm_qkv128, kv_full, vcol + h * HD + c * 64, row0k + key0);
      }
      for (int n = 0; n < nq; ++n) {
        const int st = n % QST;
        const int qs = qbase + n * BQ2;
        dev::mbar_wait(&qdo_empty[st], ((n / QST) & 1) ^ 1);
        dev::mbar_arrive_expect_tx(&qdo_full[st], 2 * Lay::QT);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          dev::tma_load_2d(sQ + st * Lay::QT + c * CHUNK64, &tm_qkv64, &qdo_full[st], h * HD + c * 64, row0 + qs);
          dev::tma_load_2d(sDO + st * Lay::QT + c * CHUNK64, &tm_do64, &qdo_full[st], h * HD + c * 64, row0 + qs);
        }
      }
    }
  } else if (warp == 1) {
    // the whole warp runs the issue loop (converged, uniform state); one elected lane issues
    {
      const uint32_t id_s = dev::make_idesc_bf16(128, BQ2, 0, 0);
      const uint32_t id_kv = dev::make_idesc_bf16(128, HD, 0, 1);
      const uint32_t id_dq = dev::make_idesc_bf16(HD, BQ2, 1, 1);
      // Descriptor bases built once; a K step only moves the 16-byte address field, so each MMA
      // costs one add instead of a descriptor rebuild (the issue rate matters at N = 64).
      const uint64_t dK_k = dev::make_sdesc_sw128(dev::smem_u32(sK), 16, 1024);
      const uint64_t dK_mn = dev::make_sdesc_sw128(dev::smem_u32(sK), CHUNK, 1024);
      const uint64_t dV_k = dev::make_sdesc_sw128(dev::smem_u32(sV), 16, 1024);
      const uint64_t dQ_k = dev::make_sdesc_sw128(dev::smem_u32(sQ), 16, 1024);
      const uint64_t dQ_mn = dev::make_sdesc_sw128(dev::smem_u32(sQ), CHUNK64, 1024);
      const uint64_t dDO_k = dev::make_sdesc_sw128(dev::smem_u32(sDO), 16, 1024);
      const uint64_t dDO_mn = dev::make_sdesc_sw128(dev::smem_u32(sDO), CHUNK64, 1024);
      const uint64_t dPt_k = dev::make_sdesc_sw128(dev::smem_u32(sPt), 16, 1024);
      const uint64_t dDSt_k = dev::make_sdesc_sw128(dev::smem_u32(sDSt), 16, 1024);
      const uint64_t dDSt_mn = dev::make_sdesc_sw128(dev::smem_u32(sDSt), CHUNK, 1024);
      constexpr uint32_t QT16 = Lay::QT >> 4;
      auto k128 = [](int kk) { return static_cast<uint64_t>((kk >> 2) * (CHUNK >> 4) + (kk & 3) * 2); };
      auto k64 = [](int kk) { return static_cast<uint64_t>((kk >> 2) * (CHUNK64 >> 4) + (kk & 3) * 2); };
      auto mn = [](int kk) { return static_cast<uint64_t>(kk * 128); };
      dev::mbar_wait(kv_full, 0);
      if (lane == 0) ATTN_TR(4002);
      auto issue_s = [&](int n) {
        const int st = n & 1, qst = n % QST;
        dev::mbar_wait(&qdo_full[qst], (n / QST) & 1);
        if (lane == 0 && n < 64) ATTN_TR(n * 16 + 0);
        if (n >= 2) dev::mbar_wait(&s_free[st], ((n - 2) >> 1) & 1);
        dev::tc_fence_after();
        if (lane == 0 && n < 64) ATTN_TR(n * 16 + 1);
        const uint64_t q_k = dQ_k + qst * QT16, do_k = dDO_k + qst * QT16;
        if (dev::elect_one_sync()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            dev::umma_f16_ss(t_s + st * BQ2, dK_k + k128(kk), q_k + k64(kk), id_s, kk > 0 ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            dev::umma_f16_ss(t_dp + st * BQ2, dV_k + k128(kk), do_k + k64(kk), id_s, kk > 0 ? 1u : 0u);
          dev::umma_commit(&s_full[st]);
        }
        __syncwarp();
      };
      issue_s(0);
      for (int n = 0; n < nq; ++n) {
        const int st = n & 1, qst = n % QST;
        if (n + 1 < nq) issue_s(n + 1);
        dev::mbar_wait(p_full, n & 1);
        dev::tc_fence_after();
        if (lane == 0 && n < 64) ATTN_TR(n * 16 + 2);
        const uint64_t q_mn = dQ_mn + qst * QT16, do_mn = dDO_mn + qst * QT16;
        if (dev::elect_one_sync()) {
          if (ts) {
            // P^T / dS^T were written into the first 32 columns of S^T_n / dP^T_n (bf16 pairs):
            // dV and dK read A from tensor memory (no shared-memory A traffic); dQ^T then
            // overwrites S^T_n, after dV has read it (MMAs execute in issue order)
#pragma unroll
            for (int kk = 0; kk < BQ2 / 16; ++kk)
              dev::umma_f16_ts(t_dv, t_s + st * BQ2 + kk * 8, do_mn + mn(kk), id_kv, (n > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < BQ2 / 16; ++kk)
              dev::umma_f16_ts(t_dk, t_dp + st * BQ2 + kk * 8, q_mn + mn(kk), id_kv, (n > 0 || kk > 0) ? 1u : 0u);
            if (ds_out == nullptr) {
#pragma unroll
              for (int kk = 0; kk < 128 / 16; ++kk)
                dev::umma_f16_ss(t_s + st * BQ2, dK_mn + mn(kk), dDSt_mn + mn(kk), id_dq, kk > 0 ? 1u : 0u);
            }
            dev::umma_commit(&dq_full[st]);  // ds_out: dV / dK have read P^T / dS^T
          } else {
          // dQ^T first (default): its TMEM drain (dQ warpgroup) then overlaps dV / dK, so the S
          // buffer it occupies is free again by the time S_{n+2} is issued
          if (dq_first) {
#pragma unroll
            for (int kk = 0; kk < 128 / 16; ++kk)
              dev::umma_f16_ss(t_s + st * BQ2, dK_mn + mn(kk), dDSt_mn + mn(kk), id_dq, kk > 0 ? 1u : 0u);
            dev::umma_commit(&dq_full[st]);
          }
#pragma unroll
          for (int kk = 0; kk < BQ2 / 16; ++kk)
            dev::umma_f16_ss(t_dv, dPt_k + k128(kk), do_mn + mn(kk), id_kv, (n > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < BQ2 / 16; ++kk)
            dev::umma_f16_ss(t_dk, dDSt_k + k128(kk), q_mn + mn(kk), id_kv, (n > 0 || kk > 0) ? 1u : 0u);
          if (!dq_first) {
#pragma unroll
            for (int kk = 0; kk < 128 / 16; ++kk)
              dev::umma_f16_ss(t_s + st * BQ2, dK_mn + mn(kk), dDSt_mn + mn(kk), id_dq, kk > 0 ? 1u : 0u);
            dev::umma_commit(&dq_full[st]);
          }
          }
          dev::umma_commit(mma_done);
          dev::umma_commit(&qdo_empty[qst]);
          if (n == nq - 1) dev::umma_commit(acc_done);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4 && warp < 12) {
    const int wg = (static_cast<int>(warp) - 4) >> 2;             // query columns [32*wg, 32*wg+32)
    const int t = static_cast<int>(warp & 3) * 32 + static_cast<int>(lane);  // key row
    const int tid = static_cast<int>(threadIdx.x) - 128;         // 0..255
    const int key = key0 + t;
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const float log2e = 1.4426950408889634f;
    // stats in the form the packed math wants: -lse (log2 units) and -scale * delta. The next
    // block's raw value is loaded one iteration ahead and only scaled when it is stored, so no
    // instruction waits on that global load until a whole block later.
    const float stat_mul = tid < BQ2 ? -log2e : -scale;
    const float* stat_src = (tid < BQ2 ? lse : delta) + static_cast<int64_t>(bh) * T;
    auto load_stat = [&](int n) -> float {
      const int qq = qbase + n * BQ2 + (tid & (BQ2 - 1));
      return (n < nq && tid < 2 * BQ2 && qq < T) ? __ldg(stat_src + qq) : 0.f;
    };
    float stat_next = load_stat(0);
    for (int n = 0; n < nq; ++n) {
      const int st = n & 1;
      const int qs = qbase + n * BQ2;
      float* st_lse = sStat + st * 2 * BQ2;
      float* st_del = st_lse + BQ2;
      if (tid < 2 * BQ2) st_lse[tid] = stat_next * stat_mul;  // [lse | delta] are contiguous
      stat_next = load_stat(n + 1);
      if (lane == 0 && (warp == 4 || warp == 8) && n < 64) ATTN_TR(n * 16 + 3 + (warp == 8) * 5);
      asm volatile("bar.sync 1, 256;" ::: "memory");
      dev::mbar_wait(&s_full[st], (n >> 1) & 1);
      dev::tc_fence_after();
      if (lane == 0 && (warp == 4 || warp == 8) && n < 64) ATTN_TR(n * 16 + 4 + (warp == 8) * 5);
      uint32_t sv[32], pv[32];
      dev::tmem_ld_32x32b_x32(t_s + lane_base + st * BQ2 + wg * 32, sv);
      dev::tmem_ld_32x32b_x32(t_dp + lane_base + st * BQ2 + wg * 32, pv);
      dev::tmem_ld_wait();
      // masks only where the block touches the diagonal or the sequence end (block-uniform)
      const bool masked = (causal && qs < key0 + 128) || qs + BQ2 > T || key0 + 128 > Tk;
      const float4* nl4 = reinterpret_cast<const float4*>(st_lse + wg * 32);
      const float4* nd4 = reinterpret_cast<const float4*>(st_del + wg * 32);
      const float2 sl2 = make_float2(scale_log2, scale_log2), sc2 = make_float2(scale, scale);
      uint32_t pk[16], dk[16];
      // the bias and mask variants are separate straight-line copies of the loop: a branch per
      // pair would split it into basic blocks and serialise each pair's exp2 latency
      auto math = [&](auto kLut, auto kMask) {
#pragma unroll
        for (int g4 = 0; g4 < 8; ++g4) {  // 4 query columns per step: P = 2^(s*sl - lse), dS = P*(dP*sc - sc*delta)
          const float4 nl = nl4[g4], nd = nd4[g4];
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int e = 2 * g4 + hh;
            float2 a = dev::ffma2(make_float2(__uint_as_float(sv[2 * e]), __uint_as_float(sv[2 * e + 1])), sl2,
                                  hh ? make_float2(nl.z, nl.w) : make_float2(nl.x, nl.y));
            if (decltype(kLut)::value && lut_h != nullptr) {  // + bias(key - query) in log2 units
              // clamped: entries past the sequence end (masked below) must still load in bounds
              const int bi = max(key + T - 1 - (qs + wg * 32 + 2 * e), 1);
              const float b0 = key < T ? __ldg(lut_h + bi) : 0.f, b1 = key < T ? __ldg(lut_h + bi - 1) : 0.f;
              a = dev::ffma2(make_float2(b0, b1), make_float2(1.4426950408889634f, 1.4426950408889634f), a);
            }
            float p0 = dev::ex2_approx(a.x), p1 = dev::ex2_approx(a.y);
            if (decltype(kMask)::value && masked) {
              const int qq = qs + wg * 32 + 2 * e;
              p0 = (qq < T && key < Tk && (!causal || qq >= key)) ? p0 : 0.f;
              p1 = (qq + 1 < T && key < Tk && (!causal || qq + 1 >= key)) ? p1 : 0.f;
            }
            const float2 t = dev::ffma2(make_float2(__uint_as_float(pv[2 * e]), __uint_as_float(pv[2 * e + 1])), sc2,
                                        hh ? make_float2(nd.z, nd.w) : make_float2(nd.x, nd.y));
            const float2 d = dev::fmul2(make_float2(p0, p1), t);
            pk[e] = dev::pack_bf16x2(p0, p1);
            dk[e] = dev::pack_bf16x2(d.x, d.y);
          }
        }
      };
      if (lut_h == nullptr && !masked) {
        math(std::false_type{}, std::false_type{});
      } else if (!masked) {  // T5: the relative-position bias on every block, the mask on few
        math(std::true_type{}, std::false_type{});
      } else {
        math(std::true_type{}, std::true_type{});  // both guards are exact no-ops when off
      }
      // sPt / sDSt were last read by block n-1's dV / dK / dQ MMAs
      if (lane == 0 && (warp == 4 || warp == 8) && n < 64) ATTN_TR(n * 16 + 5 + (warp == 8) * 5);
      // (ts with ds_out writes no shared-memory tile here: P^T / dS^T go to this block's own TMEM
      // columns, so nothing waits for block n-1's MMAs)
      if (n >= 1 && !(ts && ds_out != nullptr)) dev::mbar_wait(mma_done, (n - 1) & 1);
      if (dlut && n >= 1) dev::mbar_wait(ds_read, (n - 1) & 1);  // bias-gradient reads of dS^T_{n-1}
      if (lane == 0 && (warp == 4 || warp == 8) && n < 64) ATTN_TR(n * 16 + 6 + (warp == 8) * 5);
      if (ts) {
        // S^T_n / dP^T_n are in registers already: their first 32 columns take P^T / dS^T
        // (bf16 pairs, this warpgroup's 32 queries = 16 columns); dS^T also goes to shared
        // memory as the B operand of dQ^T
        dev::tmem_st_32x32b_x16(t_s + lane_base + st * BQ2 + wg * 16, pk);
        dev::tmem_st_32x32b_x16(t_dp + lane_base + st * BQ2 + wg * 16, dk);
        if (ds_out == nullptr) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            dev::st_sw128(sDSt, 128, t, 0, wg * 4 + u, make_uint4(dk[4 * u], dk[4 * u + 1], dk[4 * u + 2], dk[4 * u + 3]));
        }
        dev::tmem_st_wait();
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          dev::st_sw128(sPt, 128, t, 0, wg * 4 + u, make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]));
          dev::st_sw128(sDSt, 128, t, 0, wg * 4 + u, make_uint4(dk[4 * u], dk[4 * u + 1], dk[4 * u + 2], dk[4 * u + 3]));
        }
      }
      dev::fence_proxy_async_smem();
      dev::tc_fence_before();
      dev::mbar_arrive(p_full);
      if (lane == 0 && (warp == 4 || warp == 8) && n < 64) ATTN_TR(n * 16 + 7 + (warp == 8) * 5);
      if (lane == 0 && n < 64 && static_cast<int>(blockIdx.x) == trace_cta)  // the last softmax warp's arrival
        atomicMax(&g_attn_trace[n * 16 + 15], static_cast<unsigned long long>(clock64()));
    }
    // dK, dV (lane = key row) -> bf16 rows of dqkv; each warpgroup writes HD/2 columns
    dev::mbar_wait(acc_done, 0);
    dev::tc_fence_after();
    if (lane == 0 && warp == 4) ATTN_TR(4003);
    bf16* dk_row = dkv + (static_cast<int64_t>(row0k) + key) * ld_dkv + h * HD;
    bf16* dv_row = dk_row + dvoff;
#pragma unroll 1
    for (int c = wg * (HD / 64); c < (wg + 1) * (HD / 64); ++c) {
      uint32_t a[32], v[32];
      dev::tmem_ld_32x32b_x32(t_dk + lane_base + c * 32, a);
      dev::tmem_ld_32x32b_x32(t_dv + lane_base + c * 32, v);
      dev::tmem_ld_wait();
      if (key < Tk) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint4 w, z;
          w.x = dev::pack_bf16x2(__uint_as_float(a[8 * u + 0]), __uint_as_float(a[8 * u + 1]));
          w.y = dev::pack_bf16x2(__uint_as_float(a[8 * u + 2]), __uint_as_float(a[8 * u + 3]));
          w.z = dev::pack_bf16x2(__uint_as_float(a[8 * u + 4]), __uint_as_float(a[8 * u + 5]));
          w.w = dev::pack_bf16x2(__uint_as_float(a[8 * u + 6]), __uint_as_float(a[8 * u + 7]));
          z.x = dev::pack_bf16x2(__uint_as_float(v[8 * u + 0]), __uint_as_float(v[8 * u + 1]));
          z.y = dev::pack_bf16x2(__uint_as_float(v[8 * u + 2]), __uint_as_float(v[8 * u + 3]));
          z.z = dev::pack_bf16x2(__uint_as_float(v[8 * u + 4]), __uint_as_float(v[8 * u + 5]));
          z.w = dev::pack_bf16x2(__uint_as_float(v[8 * u + 6]), __uint_as_float(v[8 * u + 7]));
          *reinterpret_cast<uint4*>(dk_row + c * 32 + 8 * u) = w;
          *reinterpret_cast<uint4*>(dv_row + c * 32 + 8 * u) = z;
        }
      }
      if (colsum != nullptr && key - static_cast<int>(lane) < T) {  // k / v bias gradients of this warp's 32 keys
        float xk[32], xv[32];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float2 fk = dev::unpack_bf16x2(dev::pack_bf16x2(__uint_as_float(a[i]), __uint_as_float(a[i + 1])));
          const float2 fv = dev::unpack_bf16x2(dev::pack_bf16x2(__uint_as_float(v[i]), __uint_as_float(v[i + 1])));
          const bool in = key < T;
          xk[i] = in ? fk.x : 0.f;
          xk[i + 1] = in ? fk.y : 0.f;
          xv[i] = in ? fv.x : 0.f;
          xv[i + 1] = in ? fv.y : 0.f;
        }
        const float sk = warp_colsum32(xk, lane), sv = warp_colsum32(xv, lane);
        float* dst = colsum + static_cast<int64_t>((row0 + key - static_cast<int>(lane)) >> 5) * (3LL * Dl) + Dl +
                     h * HD + c * 32 + lane;
        dst[0] = sk;
        dst[Dl] = sv;
      }
    }
  } else if (warp >= 12) {
    // dQ^T_n: lane = head dim d, 64 query columns -> SW128 staging [4 boxes][64 rows][32 fp32]
    // (a warp writes one 128-byte row per query: conflict-free) -> TMA reduce-add
    const int d = static_cast<int>(warp & 3) * 32 + static_cast<int>(lane);
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int wd = d & 31;
    uint8_t* bx = sDQ + (d >> 5) * (BQ2 * 128);
    const bool leader = (warp == 12 && lane == 0);
    const int tq = static_cast<int>(threadIdx.x) - 384;  // 0..127: owner of bias-gradient slots == tq mod 128
    if (dlut) {
      for (int i = tq; i < T + 128; i += 128) sAcc[i] = 0.f;
    }
    if (ds_out != nullptr) {
      // dS^T_n (bf16 pairs in the first 32 columns of dP^T_n, lane = key row) -> SW128 image in
      // the (otherwise unused) dQ staging buffer, 2 x 16 KiB -> one bulk store per block
      const int tk = static_cast<int>(warp & 3) * 32 + static_cast<int>(lane);
      for (int n = 0; n < nq; ++n) {
        const int st = n & 1;
        dev::mbar_wait(&dq_full[st], (n >> 1) & 1);
        dev::tc_fence_after();
        uint32_t r[32];
        dev::tmem_ld_32x32b_x32(t_dp + lane_base + st * BQ2, r);
        dev::tmem_ld_wait();
        dev::tc_fence_before();
        dev::mbar_arrive(&s_free[st]);
        uint8_t* stg = sDQ + st * (BQ2 * 256);
        if (leader && n >= 2) dev::bulk_wait_read_1();  // block n-2's store has read this buffer
        asm volatile("bar.sync 2, 128;" ::: "memory");
#pragma unroll
        for (int u = 0; u < 8; ++u)
          dev::st_sw128(stg, 128, tk, 0, u, make_uint4(r[4 * u], r[4 * u + 1], r[4 * u + 2], r[4 * u + 3]));
        dev::fence_proxy_async_smem();
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (leader) {
          dev::bulk_store(ds_out + ds_chunk(bh, kb, n, T) * (BQ2 * 256), stg, BQ2 * 256);
          dev::bulk_commit();
        }
      }
    }
    for (int n = 0; n < (ds_out != nullptr ? 0 : nq); ++n) {
      const int st = n & 1;
      const int qs = qbase + n * BQ2;
      dev::mbar_wait(&dq_full[st], (n >> 1) & 1);
      dev::tc_fence_after();
      if (leader && n < 64) ATTN_TR(n * 16 + 13);
      uint32_t v[64];
      dev::tmem_ld_32x32b_x32(t_s + lane_base + st * BQ2, *reinterpret_cast<uint32_t(*)[32]>(v));
      dev::tmem_ld_32x32b_x32(t_s + lane_base + st * BQ2 + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
      dev::tmem_ld_wait();
      dev::tc_fence_before();
      dev::mbar_arrive(&s_free[st]);
      if (dlut) {
        // bias gradient: sums of dS^T_n (bf16 tile, [128 keys][64 queries], SW128) along the
        // diagonals key - query = const; slot key - query + T - 1 - key0 = dl + c is owned by
        // thread (dl + c) mod 128, so no two threads ever add to the same slot
        const int c = T - 1 - qs;
        const int dl0 = (((tq - c) % 128) + 128) % 128;
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
          const int dl = pass == 0 ? dl0 : dl0 - 128;
          if (pass == 1 && dl < -(BQ2 - 1)) break;
          const int e0 = dl < 0 ? -dl : 0, e1 = 127 - dl < BQ2 - 1 ? 127 - dl : BQ2 - 1;
          float acc = 0.f;
          for (int e = e0; e <= e1; ++e) {
            const int tk = e + dl;
            const uint8_t* pe = sDSt + tk * 128 + ((((e >> 3) ^ (tk & 7))) << 4) + (e & 7) * 2;
            acc += __bfloat162float(*reinterpret_cast<const bf16*>(pe));
          }
          sAcc[dl + c] += acc;
        }
        dev::mbar_arrive(ds_read);
      }
      if (leader && n < 64) ATTN_TR(n * 16 + 14);
      // the previous block's reduce-adds must have read the staging tile
      if (leader) dev::bulk_wait_read();
      asm volatile("bar.sync 2, 128;" ::: "memory");
#pragma unroll
      for (int q = 0; q < BQ2; ++q) {
        *reinterpret_cast<uint32_t*>(bx + q * 128 + (((wd >> 2) ^ (q & 7)) << 4) + (wd & 3) * 4) = v[q];
      }
      dev::fence_proxy_async_smem();
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (leader) {
#pragma unroll
        for (int bb = 0; bb < HD / 32; ++bb)
          dev::tma_reduce_add_2d(&tm_dq, sDQ + bb * (BQ2 * 128), h * HD + bb * 32, row0 + qs);
        dev::bulk_commit();
      }
    }
    if (leader) dev::bulk_wait_all();
    if (dlut) {
      float* dl_h = dlut + static_cast<int64_t>(h) * (2 * T + 128) + key0;
      for (int i = tq; i < T + 128; i += 128) {
        if (sAcc[i] != 0.f) atomicAdd(dl_h + i, sAcc[i]);
      }
    }
  }
  dev::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) ATTN_TR(4004);
  if (warp == 2) {
    dev::tc_fence_after();
    dev::tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------------------------------------
// dQ of the causal backward (head_dim 128), one CTA per (128-query tile, batch*head), heaviest
// tiles first: dQ = sum over key blocks kb <= qi of dS_(qi,kb) K_kb, accumulated in tensor memory
// (fp32, lane = query) in key order, so dQ is deterministic and never round-trips HBM in fp32.
//   warp 0      loads 64-key steps into a 3-stage ring: the two [64 keys x 64 queries] halves of
//               the dS^T tile (bulk copies of attn_bwd_tc2's SW128 images) and K [64 keys x 128]
//               (TMA, two 64-column boxes)
//   warp 1      MMA: D[128 q x 128 d] += dS (A, MN-major) K (B, MN-major), 4 k steps per stage
//   warps 2-5   epilogue: bf16 q columns of dqkv + the q bias gradient's per-32-row partials
// ---------------------------------------------------------------------------------------------
constexpr int DQ_STAGES = 3;
constexpr int DQ_STAGE = 32768;
constexpr int DQ_SMEM = DQ_STAGES * DQ_STAGE + 1024 + 128;

__global__ void __launch_bounds__(192, 2)
    attn_bwd_dq(const __grid_constant__ CUtensorMap tm_qkv64, const uint8_t* __restrict__ ds, bf16* __restrict__ dqkv,
                float* __restrict__ colsum, int T, int Hl, int nbh, int group) {
  constexpr int HD = 128;
  extern __shared__ uint8_t dq_smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dq_smem_raw) + 1023) &
                                           ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + DQ_STAGES * DQ_STAGE);
  uint64_t* empty = full + DQ_STAGES;
  uint64_t* tfull = empty + DQ_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  const int nb = T / 128;
  int unit, bh;
  work_item(static_cast<int>(blockIdx.x), nb, nbh, group, unit, bh);
  const int qi = nb - 1 - unit;  // unit 0 = the last query tile (most key blocks)
  const int b = bh / Hl, h = bh % Hl;
  const int Dl = Hl * HD;
  const int row0 = b * T;
  const int nsteps = 2 * (qi + 1);
  const uint32_t warp = dev::warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&tm_qkv64);
    for (int i = 0; i < DQ_STAGES; ++i) {
      dev::mbar_init(&full[i], 1);
      dev::mbar_init(&empty[i], 1);
    }
    dev::mbar_init(tfull, 1);
    dev::fence_barrier_init();
  }
  if (warp == 2) dev::tmem_alloc<128>(tmem_slot);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < nsteps; ++s) {
        const int st = s % DQ_STAGES, kb = s >> 1, half = s & 1;
        dev::mbar_wait(&empty[st], ((s / DQ_STAGES) & 1) ^ 1);
        dev::mbar_arrive_expect_tx(&full[st], DQ_STAGE);
        uint8_t* dst = sm + st * DQ_STAGE;
        // queries of tile qi = chunks 2 (qi - kb) and 2 (qi - kb) + 1 of key block kb
        const uint8_t* src = ds + ds_chunk(bh, kb, 2 * (qi - kb), T) * 16384 + half * 8192;
        dev::bulk_load(dst, src, 8192, &full[st]);
        dev::bulk_load(dst + 8192, src + 16384, 8192, &full[st]);
        const int krow = row0 + kb * 128 + half * 64;
        dev::tma_load_2d(dst + 16384, &tm_qkv64, &full[st], Dl + h * HD, krow);
        dev::tma_load_2d(dst + 24576, &tm_qkv64, &full[st], Dl + h * HD + 64, krow);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = dev::make_idesc_bf16(128, HD, 1, 1);
    for (int s = 0; s < nsteps; ++s) {
      const int st = s % DQ_STAGES;
      dev::mbar_wait(&full[st], (s / DQ_STAGES) & 1);
      dev::tc_fence_after();
      const uint32_t a = dev::smem_u32(sm + st * DQ_STAGE);
      if (dev::elect_one_sync()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          dev::umma_f16_ss(tmem, dev::make_sdesc_sw128(a + kk * 2048, 8192, 1024),
                           dev::make_sdesc_sw128(a + 16384 + kk * 2048, 8192, 1024), idesc,
                           (s > 0 || kk > 0) ? 1u : 0u);
        dev::umma_commit(&empty[st]);
        if (s == nsteps - 1) dev::umma_commit(tfull);
      }
      __syncwarp();
    }
  } else {
    const uint32_t q = warp & 3;  // TMEM lane quarter of this warp
    const int r32 = qi * 128 + static_cast<int>(q) * 32;  // first query of the warp's 32 rows
    dev::mbar_wait(tfull, 0);
    dev::tc_fence_after();
    bf16* out = dqkv + static_cast<int64_t>(row0 + r32 + static_cast<int>(lane)) * 3 * Dl + h * HD;
#pragma unroll 1
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t v[32];
      dev::tmem_ld_32x32b_x32(tmem + ((q * 32) << 16) + c * 32, v);
      dev::tmem_ld_wait();
      uint32_t w[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) w[i] = dev::pack_bf16x2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
#pragma unroll
      for (int u = 0; u < 4; ++u)
        *reinterpret_cast<uint4*>(out + c * 32 + 8 * u) = make_uint4(w[4 * u], w[4 * u + 1], w[4 * u + 2], w[4 * u + 3]);
      if (colsum != nullptr) {  // q bias gradient: column sums of the rounded values over the 32 rows
        float x[32];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 f = dev::unpack_bf16x2(w[i]);
          x[2 * i] = f.x;
          x[2 * i + 1] = f.y;
        }
        const float sum = warp_colsum32(x, lane);
        colsum[static_cast<int64_t>((row0 + r32) >> 5) * (3LL * Dl) + h * HD + c * 32 + lane] = sum;
      }
    }
  }
  dev::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    dev::tc_fence_after();
    dev::tmem_dealloc<128>(tmem);
  }
}

// delta[bh, q] = sum_c dO[q, c] * O[q, c]: hd/8 lanes per (row, head), 16-byte loads
__global__ void delta_kernel(const bf16* __restrict__ o, const bf16* __restrict__ dout, float* __restrict__ delta,
                             int T, int Hl, int hd, int64_t rows) {
  const int lpr = hd / 8;  // lanes per (row, head): 16 at hd = 128
  const int64_t item = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / lpr;
  const int sub = static_cast<int>(threadIdx.x % lpr);
  const bool active = item < rows * Hl;
  float s = 0.f;
  if (active) {
    const int64_t m = item / Hl;
    const int h = static_cast<int>(item % Hl);
    const int64_t off = m * (static_cast<int64_t>(Hl) * hd) + h * hd + sub * 8;
    const uint4 a = *reinterpret_cast<const uint4*>(o + off);
    const uint4 b = *reinterpret_cast<const uint4*>(dout + off);
    const uint32_t aa[4] = {a.x, a.y, a.z, a.w}, bb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 x = dev::unpack_bf16x2(aa[e]), y = dev::unpack_bf16x2(bb[e]);
      s = fmaf(x.x, y.x, fmaf(x.y, y.y, s));
    }
  }
  for (int x = lpr / 2; x > 0; x >>= 1) s += __shfl_xor_sync(0xffffffffu, s, x);
  if (active && sub == 0) {
    const int64_t m = item / Hl;
    const int h = static_cast<int>(item % Hl);
    const int64_t b2 = m / T, t = m % T;
    delta[(b2 * Hl + h) * T + t] = s;
  }
}

// scalar fallback for head dims that are not a multiple of 8 lanes' worth (one warp per row)
__global__ void delta_any_kernel(const bf16* __restrict__ o, const bf16* __restrict__ dout, float* __restrict__ delta,
                                 int T, int Hl, int hd, int64_t rows) {
  const int64_t wid = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= rows * Hl) return;
  const int64_t m = wid / Hl;
  const int h = static_cast<int>(wid % Hl);
  const int64_t off = m * (static_cast<int64_t>(Hl) * hd) + h * hd;
  float s = 0.f;
  for (int c = lane * 2; c < hd; c += 64) {
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(o + off + c));
    const float2 bb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(dout + off + c));
    s += a.x * bb.x + a.y * bb.y;
  }
#pragma unroll
  for (int x = 16; x > 0; x >>= 1) s += __shfl_xor_sync(0xffffffffu, s, x);
  if (lane == 0) {
    const int64_t b = m / T, t = m % T;
    delta[(b * Hl + h) * T + t] = s;
  }
}

void launch_delta(const bf16* o, const bf16* dout, float* delta, int T, int Hl, int hd, int64_t M, cudaStream_t s) {
  if (hd % 8 == 0 && hd / 8 <= 32 && (hd / 8 & (hd / 8 - 1)) == 0) {
    const int64_t threads = M * Hl * (hd / 8);
    delta_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(o, dout, delta, T, Hl, hd, M);
  } else {
    const int64_t warps = M * Hl;
    delta_any_kernel<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, s>>>(o, dout, delta, T, Hl, hd, M);
  }
}

// dQ (fp32 accumulator) -> bf16 q columns of dqkv, plus the q bias gradient's per-32-row column
// partials colsum[r / 32][c] of the rounded values: CTA = 32 rows x 1024 columns, 4 per thread
__global__ void __launch_bounds__(256) dq_to_bf16_colsum(const float* __restrict__ acc, bf16* __restrict__ dqkv,
                                                         int64_t rows, int Dl, float* __restrict__ colsum) {
  const int c = (blockIdx.y * 256 + threadIdx.x) * 4;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32;
  if (c >= Dl) return;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll 8
  for (int i = 0; i < 32; ++i) {
    const int64_t r = r0 + i;
    if (r < rows) {
      const float4 v = *reinterpret_cast<const float4*>(acc + r * Dl + c);
      uint2 w;
      w.x = dev::pack_bf16x2(v.x, v.y);
      w.y = dev::pack_bf16x2(v.z, v.w);
      *reinterpret_cast<uint2*>(dqkv + r * 3LL * Dl + c) = w;
      const float2 a = dev::unpack_bf16x2(w.x), b = dev::unpack_bf16x2(w.y);
      s0 += a.x;
      s1 += a.y;
      s2 += b.x;
      s3 += b.y;
    }
  }
  *reinterpret_cast<float4*>(colsum + blockIdx.x * 3LL * Dl + c) = make_float4(s0, s1, s2, s3);
}

__global__ void dq_to_bf16(const float* __restrict__ acc, bf16* __restrict__ dqkv, int64_t rows, int Dl,
                           int64_t ld_out = 0) {
  const int64_t ld = ld_out > 0 ? ld_out : 3LL * Dl;  // default: the q columns of fused dq|dk|dv rows
  const int64_t n4 = rows * Dl / 4;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n4;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = (e * 4) / Dl, c = (e * 4) % Dl;
    const float4 v = reinterpret_cast<const float4*>(acc)[e];
    uint2 w;
    w.x = dev::pack_bf16x2(v.x, v.y);
    w.y = dev::pack_bf16x2(v.z, v.w);
    *reinterpret_cast<uint2*>(dqkv + r * ld + c) = w;
  }
}

bool bwd2_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SW_ATTN_BWD_V1");
    return !(e != nullptr && e[0] == '1');
  }();
  return on;
}

// kv == nullptr: self-attention over fused q|k|v rows (gradients into the fused dqkv rows);
// otherwise cross-attention: q [B*T, ldq], k|v [B*Tk, ldkv] (v at +voff), dq [B*T, ld_dq],
// dk|dv [B*Tk, ld_dkv] (dv at +voff)
bool launch_bwd2(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, bf16* dqkv, float* scratch,
                 int B, int T, int Hl, cudaStream_t s, int causal = 1, const float* lut = nullptr,
                 float* dlut = nullptr, float scale_arg = 0.f, bool delta_ready = false,
                 float* colsum = nullptr, bool* colsum_done = nullptr, const bf16* kv = nullptr, int Tk = 0,
                 int64_t ldq = 0, int64_t ldkv = 0, int voff = 0, bf16* dkv = nullptr, int64_t ld_dq = 0,
                 int64_t ld_dkv = 0, bool allow_ds = false) {
  constexpr int HD = 128;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(attn_bwd_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize, Bwd2Layout::BYTES) !=
            cudaSuccess ||
        cudaFuncSetAttribute(attn_bwd_dq, cudaFuncAttributeMaxDynamicSharedMemorySize, DQ_SMEM) != cudaSuccess) {
      return false;
    }
    configured = true;
  }
  const int Dl = Hl * HD;
  const int64_t M = static_cast<int64_t>(B) * T;
  float* delta = scratch;
  float* dq = scratch + ((M * Hl + 63) / 64) * 64;
  // the decoder's causal self-attention: dS^T tiles out, dQ from attn_bwd_dq (scratch sized by
  // attention_bwd_scratch_floats)
  const bool ext = allow_ds && kv == nullptr && causal && lut == nullptr && dlut == nullptr && T % 128 == 0 &&
                   bwd_ts() && bwd_dq_ext();
  uint8_t* ds = ext ? reinterpret_cast<uint8_t*>(dq) : nullptr;
  if (!ext) cudaMemsetAsync(dq, 0, sizeof(float) * M * Dl, s);
  if (!delta_ready) launch_delta(o, dout, delta, T, Hl, HD, M, s);
  const bool cross = kv != nullptr;
  const CUtensorMap tm_qkv64 =
      cross ? make_tmap_bf16_2d(qkv, static_cast<uint64_t>(Dl), static_cast<uint64_t>(M), static_cast<uint64_t>(ldq), 64,
                                BQ2)
            : make_tmap_bf16_2d(qkv, 3ull * Dl, static_cast<uint64_t>(M), 3ull * Dl, 64, BQ2);
  const CUtensorMap tm_qkv128 =
      cross ? make_tmap_bf16_2d(kv, static_cast<uint64_t>(voff + Dl), static_cast<uint64_t>(B) * Tk,
                                static_cast<uint64_t>(ldkv), 64, 128)
            : make_tmap_bf16_2d(qkv, 3ull * Dl, static_cast<uint64_t>(M), 3ull * Dl, 64, 128);
  const CUtensorMap tm_do64 = make_tmap_bf16_2d(dout, static_cast<uint64_t>(Dl), static_cast<uint64_t>(M),
                                                static_cast<uint64_t>(Dl), 64, BQ2);
  const CUtensorMap tm_dq = make_tmap_f32_2d(dq, static_cast<uint64_t>(Dl), static_cast<uint64_t>(M),
                                             static_cast<uint64_t>(Dl), 32, BQ2);
  const int nb = ((cross ? Tk : T) + 127) / 128;
  const double scale = scale_arg > 0.f ? scale_arg : 1.0 / std::sqrt(static_cast<double>(HD));
  // bias-gradient partials need 32-row groups that never straddle two sequences
  float* cs = (colsum != nullptr && T % 32 == 0 && !cross) ? colsum : nullptr;
  attn_bwd_tc2<<<nb * B * Hl, 512, Bwd2Layout::BYTES, s>>>(
      tm_qkv64, tm_qkv128, tm_do64, tm_dq, lse, delta, dqkv, T, Hl, static_cast<float>(scale * 1.4426950408889634),
      static_cast<float>(scale), B * Hl, work_group(), trace_cta(), bwd_dq_first(), (lut || dlut) ? 1 : bwd_ts(),
      causal, lut, dlut, cs, cross ? Tk : T, cross ? 0 : Dl, cross ? voff : 2 * Dl, cross ? dkv : dqkv + Dl,
      cross ? ld_dkv : 3LL * Dl, cross ? voff : Dl, ds);
  if (ext) {
    attn_bwd_dq<<<nb * B * Hl, 192, DQ_SMEM, s>>>(tm_qkv64, ds, dqkv, cs, T, Hl, B * Hl, work_group());
  } else if (cs != nullptr) {
    dq_to_bf16_colsum<<<dim3(static_cast<unsigned>((M + 31) / 32), (Dl + 1023) / 1024), 256, 0, s>>>(dq, dqkv, M, Dl,
                                                                                                      cs);
  } else {
    dq_to_bf16<<<1184, 256, 0, s>>>(dq, dqkv, M, Dl, cross ? ld_dq : 0);
  }
  if (colsum_done != nullptr) *colsum_done = cs != nullptr;
  return true;
}

template <int HD>
bool launch_bwd(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, bf16* dqkv, float* scratch,
                int B, int T, int Hl, cudaStream_t s, bool delta_ready, float* colsum, bool* colsum_done) {
  if (HD == 128 && bwd2_enabled())
    return launch_bwd2(qkv, o, lse, dout, dqkv, scratch, B, T, Hl, s, 1, nullptr, nullptr, 0.f, delta_ready, colsum,
                       colsum_done, nullptr, 0, 0, 0, 0, nullptr, 0, 0, true);
  using Lay = BwdLayout<HD>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(attn_bwd_tc<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay::BYTES) !=
        cudaSuccess) {
      return false;
    }
    configured = true;
  }
  const int Dl = Hl * HD;
  const int64_t M = static_cast<int64_t>(B) * T;
  float* delta = scratch;
  float* dq = scratch + ((M * Hl + 63) / 64) * 64;
  cudaMemsetAsync(dq, 0, sizeof(float) * M * Dl, s);
  if (!delta_ready) launch_delta(o, dout, delta, T, Hl, HD, M, s);
  const CUtensorMap tm_qkv = make_tmap_bf16_2d(qkv, 3ull * Dl, static_cast<uint64_t>(M), 3ull * Dl, 64, 128);
  const CUtensorMap tm_do = make_tmap_bf16_2d(dout, static_cast<uint64_t>(Dl), static_cast<uint64_t>(M),
                                              static_cast<uint64_t>(Dl), 64, 128);
  const CUtensorMap tm_dq = make_tmap_f32_2d(dq, static_cast<uint64_t>(Dl), static_cast<uint64_t>(M),
                                             static_cast<uint64_t>(Dl), 32, 128);
  const int nb = (T + 127) / 128;
  const double scale = 1.0 / std::sqrt(static_cast<double>(HD));
  attn_bwd_tc<HD><<<nb * B * Hl, 384, Lay::BYTES, s>>>(tm_qkv, tm_do, tm_dq, lse, delta, dq, dqkv, T, Hl,
                                                        static_cast<float>(scale * 1.4426950408889634),
                                                        static_cast<float>(scale));
  dq_to_bf16<<<1184, 256, 0, s>>>(dq, dqkv, M, Dl);
  return true;
}

}  // namespace

void attention_hd256_trace_read(unsigned long long* out);

// SW_ATTN_TRACE_HD256=1: the head_dim-256 backward's trace (attention_hd256.cu) instead
void attention_trace_read(unsigned long long* out) {
  const char* e = std::getenv("SW_ATTN_TRACE_HD256");
  if (e != nullptr && e[0] == '1') {
    attention_hd256_trace_read(out);
    return;
  }
  cudaMemcpyFromSymbol(out, g_attn_trace, sizeof(unsigned long long) * 4096);
}

bool attention_mma_fwd_ex(const bf16* qkv, bf16* o, float* lse, int B, int T, int Hl, int hd, int causal,
                          const float* lut, float scale, cudaStream_t s) {
  if (hd != 128 || ((3 * Hl * hd) % 8) != 0) return false;
  return launch_fwd2(qkv, o, lse, B, T, Hl, s, causal, lut, scale);
}

bool attention_hd256_fwd(const bf16* qkv, bf16* o, float* lse, int B, int T, int Hl, cudaStream_t s);
bool attention_hd256_bwd(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, bf16* dqkv,
                         float* scratch, int B, int T, int Hl, cudaStream_t s, bool delta_ready);

// shared with attention_hd256.cu: delta = rowsum(dO * O) per (bh, q), and the fp32 dQ accumulator
// -> bf16 q columns of dqkv
void attn_delta(const bf16* o, const bf16* dout, float* delta, int T, int Hl, int hd, int64_t M, cudaStream_t s) {
  launch_delta(o, dout, delta, T, Hl, hd, M, s);
}
void attn_dq_to_bf16(const float* dq, bf16* dqkv, int64_t M, int Dl, cudaStream_t s) {
  dq_to_bf16<<<1184, 256, 0, s>>>(dq, dqkv, M, Dl);
}

bool attention_mma_fwd(const bf16* qkv, bf16* o, float* lse, int B, int T, int Hl, int hd, cudaStream_t s) {
  if (((3 * Hl * hd) % 8) != 0) return false;
  if (hd == 256) return attention_hd256_fwd(qkv, o, lse, B, T, Hl, s);
  if (hd == 128) {
    if (fwd2_enabled() && fwd3_enabled()) return launch_fwd3(qkv, o, lse, B, T, Hl, s);
    return fwd2_enabled() ? launch_fwd2(qkv, o, lse, B, T, Hl, s) : launch_fwd<128>(qkv, o, lse, B, T, Hl, s);
  }
  if (hd == 64) return launch_fwd<64>(qkv, o, lse, B, T, Hl, s);
  return false;
}

// Cross-attention (T5, non-causal, no bias) for head_dim 128 on the tensor cores: queries [B*Tq]
// of q (row pitch ldq), keys / values [B*Tk] of kv (k at column h*128, v at voff + h*128).
bool attention_mma_fwd_cross(const bf16* q, int64_t ldq, const bf16* kv, int64_t ldkv, int voff, bf16* o, float* lse,
                             int B, int Tq, int Tk, int Hl, int hd, float scale, cudaStream_t s) {
  if (hd != 128 || ldq % 8 != 0 || ldkv % 8 != 0 || voff % 8 != 0) return false;
  return launch_fwd2(q, o, lse, B, Tq, Hl, s, 0, nullptr, scale, kv, Tk, ldq, ldkv, voff);
}

bool attention_mma_bwd_cross(const bf16* q, int64_t ldq, const bf16* kv, int64_t ldkv, int voff, const bf16* o,
                             const float* lse, const bf16* dout, bf16* dq, int64_t ld_dq, bf16* dkv, int64_t ld_dkv,
                             float* scratch, int B, int Tq, int Tk, int Hl, int hd, float scale, cudaStream_t s) {
  if (hd != 128 || ldq % 8 != 0 || ldkv % 8 != 0 || voff % 8 != 0 || ld_dq % 4 != 0 || !bwd2_enabled()) return false;
  return launch_bwd2(q, o, lse, dout, dq, scratch, B, Tq, Hl, s, 0, nullptr, nullptr, scale, false, nullptr, nullptr,
                     kv, Tk, ldq, ldkv, voff, dkv, ld_dq, ld_dkv);
}

bool attention_mma_bwd_ex(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, bf16* dqkv,
                          float* scratch, int B, int T, int Hl, int hd, int causal, const float* lut, float* dlut,
                          float scale, cudaStream_t s) {
  if (hd != 128 || ((Hl * hd) % 8) != 0 || ((lut || dlut) && T + 128 > Bwd2Layout::PT / 4) || !bwd2_enabled())
    return false;
  return launch_bwd2(qkv, o, lse, dout, dqkv, scratch, B, T, Hl, s, causal, lut, dlut, scale);
}

int64_t attention_bwd_scratch_floats(int B, int T, int Hl, int hd) {
  const int64_t M = static_cast<int64_t>(B) * T;
  int64_t n = M * Hl + 2 * M * Hl * hd + 64;
  if (hd == 128 && T % 128 == 0) {  // delta + the dS^T tiles of attn_bwd_dq
    const int64_t ds = static_cast<int64_t>(B) * Hl * ds_chunks_before(T / 128, T) * (16384 / 4);
    n = std::max(n, (M * Hl + 63) / 64 * 64 + ds);
  }
  return n;
}

bool attention_mma_bwd(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, bf16* dqkv,
                       float* scratch, int B, int T, int Hl, int hd, cudaStream_t s, bool delta_ready,
                       float* colsum, bool* colsum_done) {
  if (((Hl * hd) % 8) != 0) return false;
  if (hd == 256) {
    if (colsum_done != nullptr) *colsum_done = false;
    return attention_hd256_bwd(qkv, o, lse, dout, dqkv, scratch, B, T, Hl, s, delta_ready);
  }
  if (hd == 128) return launch_bwd<128>(qkv, o, lse, dout, dqkv, scratch, B, T, Hl, s, delta_ready, colsum, colsum_done);
  if (hd == 64) return launch_bwd<64>(qkv, o, lse, dout, dqkv, scratch, B, T, Hl, s, delta_ready, colsum, colsum_done);
  return false;
}

}  // namespace k
}  // namespace sw
