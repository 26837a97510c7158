// tcgen05 flash attention for head_dim 256 (GPT-J-6B shape, BASELINE cfg3: H = 16, hd = 256),
// causal, head-sharded -- the same computation as attention_mma.cu's head_dim-128 kernels
// (graph.hpp:650-661 with model.hpp:100-106's causal mask) under a different TMEM budget: an fp32
// accumulator of 128 rows x 256 columns fills half of tensor memory, so the hd-128 layouts (two
// query tiles, or S^T / dP^T double buffers beside dK and dV) do not fit.
//
// Forward, one CTA per (128-query tile, batch*head), heaviest tile first, 64-key blocks:
//   warp 0     TMA producer: K_j / V_j ([64 keys x 256] each, 4 SW128 chunks) into a 3-stage ring
//   warp 1     MMA issuer:   S_j = Q K_j^T into one of two TMEM S buffers while the softmax works on
//              the other (Q is the A operand straight from TMEM: only K streams through shared
//              memory), then O += P_j V_j (P from TMEM, V as an MN-major operand)
//   warp 2     TMEM allocator (512 columns: O 256 | Q 128 | S0 64 | S1 64)
//   warps 4-7  softmax: thread = query row. Loads its Q row into TMEM once, then per block reads
//              S_j, applies the lazily kept running max (a row's max moves only when it grows by
//              more than 2^8 in exp2 units; O is rescaled in TMEM then), writes P_j (bf16) over
//              S_j, and finally O / l -> bf16 and the log-sum-exp.
//
// Backward, two passes per (128-key block, batch*head) over 64-query blocks from the diagonal on
// (lane = key row in every accumulator); each pass keeps one 128 x 256 fp32 gradient in TMEM:
//   dV pass   S^T_n = K Q_n^T (K in TMEM: only Q streams through shared memory; S^T double-
//             buffered so S^T_{n+1} runs while the softmax warpgroup turns S^T_n into P^T_n),
//             dV += P^T_n dO_n (P^T from TMEM).            TMEM: dV 256 | K 128 | S^T 2 x 64
//   dK/dQ pass S^T_n = K Q_n^T (K from shared memory), dP^T_n = V dO_n^T (V in TMEM),
//             dS^T = P^T (dP^T - delta) scale -> TMEM (A of dK) and shared memory (B of dQ),
//             dK += dS^T Q_n, dQ^T_n = K^T dS^T_n in two 128-row halves of the head dimension
//             written over S^T_n / dP^T_n, drained by a warpgroup with vector reductions into an
//             fp32 dQ accumulator.                        TMEM: dK 256 | V 128 | S^T 64 | dP^T 64
// The S^T / dP^T recompute of the second pass is the price of the budget (6 of the 5 + 1 tile
// products); the dQ accumulator is converted to bf16 once per launch (attention_mma.cu).
#include <type_traits>
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "kernels.h"
#include "sm100.cuh"
#include "tensormap.h"

namespace sw {
namespace k {
namespace {

constexpr int HD = 256;

// phase trace of one backward dK/dQ CTA (SW_ATTN_TRACE_CTA): per block n < 200, slots 16 n + ...
__device__ unsigned long long g_hd256_trace[4096];
#define T256(slot)                                                                                    \
  do {                                                                                                \
    if (static_cast<int>(blockIdx.x) == trace_cta && (slot) < 4096) g_hd256_trace[(slot)] = clock64(); \
  } while (0)
constexpr int BQ = 128;
constexpr int BK = 64;
constexpr int CH = BK * 128;  // one [64 rows x 64 bf16] SW128 chunk: 8 KiB
constexpr int NST = 3;        // K/V ring depth

struct FwdLay {
  static constexpr int KV = BK * HD * 2;  // 32 KiB per K (or V) block
  static constexpr int OFF_K = 0;                  // [NST]
  static constexpr int OFF_V = OFF_K + NST * KV;   // [NST]
  static constexpr int OFF_BAR = OFF_V + NST * KV;
  static constexpr int BYTES = OFF_BAR + 256;
};

// TMEM columns
constexpr uint32_t T_O = 0, T_Q = 256, T_S = 384;  // S buffer b at T_S + 64 b

// (batch*head) in groups of G, heaviest query tile of every head first (attention_mma.cu's order)
__device__ __forceinline__ void work_item256(int idx, int nunits, int nbh, int G, int& unit, int& bh) {
  const int grp = idx / (G * nunits);
  const int r = idx - grp * G * nunits;
  const int g = min(G, nbh - grp * G);
  unit = r / g;
  bh = grp * G + r % g;
}

__global__ void __launch_bounds__(256, 1)
    attn_fwd_hd256(const __grid_constant__ CUtensorMap tm_kv, const bf16* __restrict__ qkv, bf16* __restrict__ out,
                   float* __restrict__ lse, int T, int Hl, float scale_log2, float scale, int nbh) {
  using Lay = FwdLay;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sK = smem + Lay::OFF_K;
  uint8_t* sV = smem + Lay::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::OFF_BAR);
  uint64_t* kv_full = bars;            // [NST]
  uint64_t* kv_empty = bars + NST;     // [NST]
  uint64_t* s_full = bars + 2 * NST;   // [2]
  uint64_t* p_full = s_full + 2;       // [2]
  uint64_t* pv_done = p_full + 2;      // [2] (per block parity: never two phases behind its waiter)
  uint64_t* q_ready = pv_done + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_ready + 1);

  const int nqb = (T + BQ - 1) / BQ;
  int rank_, bh;
  work_item256(static_cast<int>(blockIdx.x), nqb, nbh, 8, rank_, bh);
  const int qi = nqb - 1 - rank_;  // heaviest (latest) query tile first
  const int b = bh / Hl, h = bh % Hl;
  const int Dl = Hl * HD;
  const int row0 = b * T;
  const int q0 = qi * BQ;
  const int nkb = min((q0 + BQ + BK - 1) / BK, (T + BK - 1) / BK);  // causal: key blocks through the diagonal

  const uint32_t warp = dev::warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&tm_kv);
    for (int i = 0; i < NST; ++i) {
      dev::mbar_init(&kv_full[i], 1);
      dev::mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      dev::mbar_init(&s_full[i], 1);
      dev::mbar_init(&p_full[i], 128);
      dev::mbar_init(&pv_done[i], 1);
    }
    dev::mbar_init(q_ready, 128);
    dev::fence_barrier_init();
  }
  if (warp == 2) dev::tmem_alloc<512>(tmem_slot);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int j = 0; j < nkb; ++j) {
        const int st = j % NST;
        dev::mbar_wait(&kv_empty[st], ((j / NST) & 1) ^ 1);
        dev::mbar_arrive_expect_tx(&kv_full[st], 2 * Lay::KV);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          dev::tma_load_2d(sK + st * Lay::KV + c * CH, &tm_kv, &kv_full[st], Dl + h * HD + c * 64, row0 + j * BK);
          dev::tma_load_2d(sV + st * Lay::KV + c * CH, &tm_kv, &kv_full[st], 2 * Dl + h * HD + c * 64, row0 + j * BK);
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t id_s = dev::make_idesc_bf16(BQ, BK, 0, 0);
    const uint32_t id_o = dev::make_idesc_bf16(BQ, HD, 0, 1);
    const uint64_t dk = dev::make_sdesc_sw128(dev::smem_u32(sK), 16, 1024);
    const uint64_t dv = dev::make_sdesc_sw128(dev::smem_u32(sV), CH, 1024);
    constexpr uint64_t KV16 = Lay::KV >> 4;
    dev::mbar_wait(q_ready, 0);
    dev::tc_fence_after();
    auto issue_s = [&](int j) {
      const int st = j % NST;
      dev::mbar_wait(&kv_full[st], (j / NST) & 1);
      dev::tc_fence_after();
      const uint64_t bk = dk + st * KV16;
      if (dev::elect_one_sync()) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)  // K step kk: Q columns [8 kk, 8 kk + 8); K chunk kk / 4, +32 B
          dev::umma_f16_ts(tmem + T_S + (j & 1) * 64, tmem + T_Q + kk * 8,
                           bk + static_cast<uint64_t>((kk >> 2) * (CH >> 4) + (kk & 3) * 2), id_s, kk > 0 ? 1u : 0u);
        dev::umma_commit(&s_full[j & 1]);
      }
      __syncwarp();
    };
    issue_s(0);
    for (int j = 0; j < nkb; ++j) {
      // S_{j+1} goes into the buffer of P_{j-1}, whose P V was issued (and so executes) before it
      if (j + 1 < nkb) issue_s(j + 1);
      dev::mbar_wait(&p_full[j & 1], (j >> 1) & 1);
      dev::tc_fence_after();
      const uint64_t bv = dv + (j % NST) * KV16;
      if (dev::elect_one_sync()) {
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)  // P (bf16 pairs) in the first 32 columns of S_j
          dev::umma_f16_ts(tmem + T_O, tmem + T_S + (j & 1) * 64 + kk * 8, bv + static_cast<uint64_t>(kk * 128), id_o,
                           (j > 0 || kk > 0) ? 1u : 0u);
        dev::umma_commit(&pv_done[j & 1]);
        dev::umma_commit(&kv_empty[j % NST]);  // K_j (read by S_j, issued earlier) and V_j consumed
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int r = static_cast<int>(warp & 3) * 32 + static_cast<int>(lane);
    const int q = q0 + r;
    const uint32_t lb = static_cast<uint32_t>((warp & 3) * 32) << 16;
    // Q row -> TMEM columns [T_Q, T_Q + 128) (bf16 pairs, the A-operand layout of a K-major tile)
    {
      const uint4* src = reinterpret_cast<const uint4*>(qkv + (static_cast<int64_t>(row0) + min(q, T - 1)) * 3LL * Dl + h * HD);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t w[32];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint4 x = q < T ? __ldg(src + c * 8 + u) : make_uint4(0, 0, 0, 0);
          w[4 * u] = x.x;
          w[4 * u + 1] = x.y;
          w[4 * u + 2] = x.z;
          w[4 * u + 3] = x.w;
        }
        dev::tmem_st_32x32b_x32(tmem + lb + T_Q + c * 32, w);
      }
      dev::tmem_st_wait();
      dev::tc_fence_before();
      dev::mbar_arrive(q_ready);
    }
    const uint32_t tO = tmem + lb + T_O;
    const float2 sl2 = make_float2(scale_log2, scale_log2);
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < nkb; ++j) {
      dev::mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      dev::tc_fence_after();
      const uint32_t tS = tmem + lb + T_S + (j & 1) * 64;
      uint32_t v[64];
      auto load_s = [&]() {
        dev::tmem_ld_32x32b_x32(tS, *reinterpret_cast<uint32_t(*)[32]>(v));
        dev::tmem_ld_32x32b_x32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        dev::tmem_ld_wait();
        if ((j + 1) * BK > q0 || (j + 1) * BK > T) {
#pragma unroll
          for (int i = 0; i < BK; ++i) {
            const int key = j * BK + i;
            if (key > q || key >= T) v[i] = __float_as_uint(-INFINITY);
          }
        }
      };
      auto rowmax = [&]() {
        float m4[4] = {__uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]), __uint_as_float(v[3])};
#pragma unroll
        for (int i = 4; i < BK; i += 8) {
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
        for (int e = 0; e < BK / 2; ++e) {
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
          dev::mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);  // every earlier P V has landed in O
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
      dev::tmem_st_32x32b_x32(tS, *reinterpret_cast<uint32_t(*)[32]>(v));
      dev::tmem_st_wait();
      dev::tc_fence_before();
      dev::mbar_arrive(&p_full[j & 1]);
    }
    dev::mbar_wait(&pv_done[(nkb - 1) & 1], ((nkb - 1) >> 1) & 1);
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
  dev::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    dev::tc_fence_after();
    dev::tmem_dealloc<512>(tmem);
  }
}

// ---------------------------------------------------------------------------------------------
// backward
// ---------------------------------------------------------------------------------------------
constexpr int BQB = 64;                 // queries per backward block
constexpr int QB = BQB * HD * 2;        // one Q (or dO) block: 32 KiB, 4 chunks of [64 rows x 128 B]
constexpr int KT = 128 * HD * 2;        // one K (or V) tile of 128 keys: 64 KiB, 4 chunks of 16 KiB
constexpr int CH128 = 128 * 128;        // [128 rows x 64 bf16] SW128 chunk

// a [128 rows x 256] bf16 row of this thread (lane = row) from global into TMEM columns
// [col, col + 128) as bf16 pairs (the A-operand layout of a K-major tile); zeros past the end
__device__ __forceinline__ void row_to_tmem(const bf16* src, bool valid, uint32_t taddr) {
  const uint4* p = reinterpret_cast<const uint4*>(src);
#pragma unroll 1
  for (int c = 0; c < 4; ++c) {
    uint32_t w[32];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint4 x = valid ? __ldg(p + c * 8 + u) : make_uint4(0, 0, 0, 0);
      w[4 * u] = x.x;
      w[4 * u + 1] = x.y;
      w[4 * u + 2] = x.z;
      w[4 * u + 3] = x.w;
    }
    dev::tmem_st_32x32b_x32(taddr + c * 32, w);
  }
  dev::tmem_st_wait();
}

// this thread's 128 x 256 fp32 accumulator row (TMEM columns [col, col + 256)) -> bf16 in global
__device__ __forceinline__ void acc_row_out(uint32_t taddr, bf16* dst, bool valid) {
#pragma unroll 1
  for (int c = 0; c < HD / 32; ++c) {
    uint32_t a[32];
    dev::tmem_ld_32x32b_x32(taddr + c * 32, a);
    dev::tmem_ld_wait();
    if (valid) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint4 w;
        w.x = dev::pack_bf16x2(__uint_as_float(a[8 * u + 0]), __uint_as_float(a[8 * u + 1]));
        w.y = dev::pack_bf16x2(__uint_as_float(a[8 * u + 2]), __uint_as_float(a[8 * u + 3]));
        w.z = dev::pack_bf16x2(__uint_as_float(a[8 * u + 4]), __uint_as_float(a[8 * u + 5]));
        w.w = dev::pack_bf16x2(__uint_as_float(a[8 * u + 6]), __uint_as_float(a[8 * u + 7]));
        *reinterpret_cast<uint4*>(dst + c * 32 + 8 * u) = w;
      }
    }
  }
}

// -------------------------------- dV pass --------------------------------
constexpr int DV_NST = 3;
struct DvLay {
  static constexpr int OFF_Q = 0;                     // [DV_NST]
  static constexpr int OFF_DO = OFF_Q + DV_NST * QB;  // [DV_NST]
  static constexpr int OFF_STAT = OFF_DO + DV_NST * QB;  // [2][64] -lse log2e of the block
  static constexpr int OFF_BAR = OFF_STAT + 2 * BQB * 4;
  static constexpr int BYTES = OFF_BAR + 256;
};
constexpr uint32_t D_ACC = 0, D_K = 256, D_S = 384;  // S^T buffer b at D_S + 64 b

__global__ void __launch_bounds__(256, 1)
    attn_bwd_hd256_dv(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                      const bf16* __restrict__ qkv, const float* __restrict__ lse, bf16* __restrict__ dqkv, int T,
                      int Hl, float scale_log2, int nbh, int trace_cta) {
  using Lay = DvLay;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sQ = smem + Lay::OFF_Q;
  uint8_t* sDO = smem + Lay::OFF_DO;
  float* sStat = reinterpret_cast<float*>(smem + Lay::OFF_STAT);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::OFF_BAR);
  uint64_t* qd_full = bars;                 // [DV_NST]
  uint64_t* qd_empty = bars + DV_NST;       // [DV_NST]
  uint64_t* s_full = bars + 2 * DV_NST;     // [2]
  uint64_t* p_full = s_full + 2;            // [2]
  uint64_t* k_ready = p_full + 2;
  uint64_t* acc_done = k_ready + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);

  const int nkb = (T + 127) / 128;
  int rank_, bh;
  work_item256(static_cast<int>(blockIdx.x), nkb, nbh, 8, rank_, bh);
  const int kb = rank_;  // key block 0 sees the most query blocks
  const int b = bh / Hl, h = bh % Hl;
  const int Dl = Hl * HD;
  const int row0 = b * T;
  const int key0 = kb * 128;
  const int nq = (T - key0 + BQB - 1) / BQB;  // causal: query blocks from the diagonal on

  const uint32_t warp = dev::warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&tm_q);
    dev::tma_prefetch_desc(&tm_do);
    for (int i = 0; i < DV_NST; ++i) {
      dev::mbar_init(&qd_full[i], 1);
      dev::mbar_init(&qd_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      dev::mbar_init(&s_full[i], 1);
      dev::mbar_init(&p_full[i], 128);
    }
    dev::mbar_init(k_ready, 128);
    dev::mbar_init(acc_done, 1);
    dev::fence_barrier_init();
  }
  if (warp == 2) dev::tmem_alloc<512>(tmem_slot);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int n = 0; n < nq; ++n) {
        const int st = n % DV_NST;
        const int qs = key0 + n * BQB;
        dev::mbar_wait(&qd_empty[st], ((n / DV_NST) & 1) ^ 1);
        dev::mbar_arrive_expect_tx(&qd_full[st], 2 * QB);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          dev::tma_load_2d(sQ + st * QB + c * CH, &tm_q, &qd_full[st], h * HD + c * 64, row0 + qs);
          dev::tma_load_2d(sDO + st * QB + c * CH, &tm_do, &qd_full[st], h * HD + c * 64, row0 + qs);
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t id_s = dev::make_idesc_bf16(128, BQB, 0, 0);
    const uint32_t id_v = dev::make_idesc_bf16(128, HD, 0, 1);
    const uint64_t dq = dev::make_sdesc_sw128(dev::smem_u32(sQ), 16, 1024);
    const uint64_t ddo = dev::make_sdesc_sw128(dev::smem_u32(sDO), CH, 1024);
    constexpr uint64_t QB16 = QB >> 4;
    dev::mbar_wait(k_ready, 0);
    dev::tc_fence_after();
    auto issue_s = [&](int n) {
      const int st = n % DV_NST;
      dev::mbar_wait(&qd_full[st], (n / DV_NST) & 1);
      dev::tc_fence_after();
      const uint64_t bq = dq + st * QB16;
      if (dev::elect_one_sync()) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          dev::umma_f16_ts(tmem + D_S + (n & 1) * 64, tmem + D_K + kk * 8,
                           bq + static_cast<uint64_t>((kk >> 2) * (CH >> 4) + (kk & 3) * 2), id_s, kk > 0 ? 1u : 0u);
        dev::umma_commit(&s_full[n & 1]);
      }
      __syncwarp();
    };
    if (lane == 0) T256(2000);
    issue_s(0);
    for (int n = 0; n < nq; ++n) {
      if (n + 1 < nq) issue_s(n + 1);  // into the buffer of P^T_{n-1}, whose dV MMA precedes it
      if (lane == 0) T256(16 * n);
      dev::mbar_wait(&p_full[n & 1], (n >> 1) & 1);
      if (lane == 0) T256(16 * n + 1);
      dev::tc_fence_after();
      const uint64_t bdo = ddo + (n % DV_NST) * QB16;
      if (dev::elect_one_sync()) {
#pragma unroll
        for (int kk = 0; kk < BQB / 16; ++kk)  // P^T (bf16 pairs) in the first 32 columns of S^T_n
          dev::umma_f16_ts(tmem + D_ACC, tmem + D_S + (n & 1) * 64 + kk * 8, bdo + static_cast<uint64_t>(kk * 128), id_v,
                           (n > 0 || kk > 0) ? 1u : 0u);
        dev::umma_commit(&qd_empty[n % DV_NST]);
        if (n == nq - 1) dev::umma_commit(acc_done);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int t = static_cast<int>(warp & 3) * 32 + static_cast<int>(lane);  // key row
    const int key = key0 + t;
    const uint32_t lb = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int64_t ld = 3LL * Dl;
    row_to_tmem(qkv + (static_cast<int64_t>(row0) + min(key, T - 1)) * ld + Dl + h * HD, key < T, tmem + lb + D_K);
    dev::tc_fence_before();
    dev::mbar_arrive(k_ready);
    const float log2e = 1.4426950408889634f;
    const float* lse_bh = lse + static_cast<int64_t>(bh) * T;
    const float2 sl2 = make_float2(scale_log2, scale_log2);
    for (int n = 0; n < nq; ++n) {
      const int qs = key0 + n * BQB;
      const bool tw = warp == 4 && lane == 0;
      // the block's -lse log2e through shared memory (double-buffered: one barrier per block),
      // loaded before the wait for S^T so the global load latency is hidden
      float* st = sStat + (n & 1) * BQB;
      if (t < BQB) st[t] = qs + t < T ? -__ldg(lse_bh + qs + t) * log2e : 0.f;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (tw) T256(16 * n + 4);
      dev::mbar_wait(&s_full[n & 1], (n >> 1) & 1);
      if (tw) T256(16 * n + 5);
      dev::tc_fence_after();
      const uint32_t tS = tmem + lb + D_S + (n & 1) * 64;
      uint32_t v[64];
      dev::tmem_ld_32x32b_x32(tS, *reinterpret_cast<uint32_t(*)[32]>(v));
      dev::tmem_ld_32x32b_x32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
      dev::tmem_ld_wait();
      const bool masked = qs < key0 + 128 || qs + BQB > T || key0 + 128 > T;
      const float2* nl2 = reinterpret_cast<const float2*>(st);
      // masked / unmasked as separate straight-line loops (a branch per pair serialises the exps)
      auto pmath = [&](auto kMask) {
#pragma unroll
        for (int e = 0; e < BQB / 2; ++e) {  // P^T = 2^(s * sl - lse * log2e)
          const int qq = qs + 2 * e;
          const float2 a = dev::ffma2(make_float2(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1])), sl2, nl2[e]);
          float p0 = dev::ex2_approx(a.x), p1 = dev::ex2_approx(a.y);
          if constexpr (decltype(kMask)::value) {
            p0 = (qq < T && key < T && qq >= key) ? p0 : 0.f;
            p1 = (qq + 1 < T && key < T && qq + 1 >= key) ? p1 : 0.f;
          }
          v[e] = dev::pack_bf16x2(p0, p1);
        }
      };
      if (masked) pmath(std::true_type{}); else pmath(std::false_type{});
      dev::tmem_st_32x32b_x32(tS, *reinterpret_cast<uint32_t(*)[32]>(v));
      dev::tmem_st_wait();
      dev::tc_fence_before();
      dev::mbar_arrive(&p_full[n & 1]);
      if (tw) T256(16 * n + 6);
    }
    if (warp == 4 && lane == 0) T256(2001);
    dev::mbar_wait(acc_done, 0);
    dev::tc_fence_after();
    acc_row_out(tmem + lb + D_ACC, dqkv + (static_cast<int64_t>(row0) + key) * ld + 2 * Dl + h * HD, key < T);
  }
  dev::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    dev::tc_fence_after();
    dev::tmem_dealloc<512>(tmem);
  }
}

// -------------------------------- dK / dQ pass --------------------------------
struct DkLay {
  static constexpr int OFF_K = 0;                 // [128 keys x 256], 4 chunks of 16 KiB
  static constexpr int OFF_Q = OFF_K + KT;        // [2]
  static constexpr int OFF_DO = OFF_Q + 2 * QB;   // [2]
  static constexpr int OFF_DS = OFF_DO + 2 * QB;  // dS^T [128 keys x 64 queries] bf16, SW128 (16 KiB)
  // dQ staging: 4 TMA boxes of [64 queries x 32 fp32]; boxes 0-1 reuse the dS^T tile (free once
  // dQ^T_n has executed), boxes 2-3 follow it
  static constexpr int OFF_DQX = OFF_DS + 128 * BQB * 2;
  static constexpr int OFF_STAT = OFF_DQX + 2 * BQB * 128;  // -lse log2e | -delta scale of the block
  static constexpr int OFF_BAR = OFF_STAT + 2 * BQB * 4;
  static constexpr int BYTES = OFF_BAR + 256;
};
constexpr uint32_t K_ACC = 0, K_V = 256, K_S = 384, K_DP = 448;

__global__ void __launch_bounds__(384, 1)
    attn_bwd_hd256_dkq(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_q,
                       const __grid_constant__ CUtensorMap tm_do, const __grid_constant__ CUtensorMap tm_dq,
                       const bf16* __restrict__ qkv,
                       const float* __restrict__ lse, const float* __restrict__ delta, bf16* __restrict__ dqkv,
                       float* __restrict__ dq, int T, int Hl, float scale_log2, float scale, int nbh, int trace_cta) {
  using Lay = DkLay;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sK = smem + Lay::OFF_K;
  uint8_t* sQ = smem + Lay::OFF_Q;
  uint8_t* sDO = smem + Lay::OFF_DO;
  uint8_t* sDS = smem + Lay::OFF_DS;
  uint8_t* sDQX = smem + Lay::OFF_DQX;
  float* sStat = reinterpret_cast<float*>(smem + Lay::OFF_STAT);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Lay::OFF_BAR);
  uint64_t* k_full = bars;
  uint64_t* qd_full = bars + 1;   // [2]
  uint64_t* qd_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;    // S^T_n and dP^T_n are in TMEM
  uint64_t* p_full = bars + 6;    // dS^T_n written (TMEM + smem)
  uint64_t* dq_full = bars + 7;   // dK += .. and dQ^T_n issued and done
  uint64_t* s_free = bars + 8;    // dQ^T_n drained: the S^T / dP^T columns may be rewritten
  uint64_t* v_ready = bars + 9;
  uint64_t* stage_free = bars + 10;  // dQ_n's staging (boxes 0-1 = the dS^T tile) has been read by TMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 11);

  const int nkb = (T + 127) / 128;
  int rank_, bh;
  work_item256(static_cast<int>(blockIdx.x), nkb, nbh, 8, rank_, bh);
  const int kb = rank_;
  const int b = bh / Hl, h = bh % Hl;
  const int Dl = Hl * HD;
  const int row0 = b * T;
  const int key0 = kb * 128;
  const int nq = (T - key0 + BQB - 1) / BQB;

  const uint32_t warp = dev::warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    dev::tma_prefetch_desc(&tm_k);
    dev::tma_prefetch_desc(&tm_q);
    dev::tma_prefetch_desc(&tm_do);
    dev::tma_prefetch_desc(&tm_dq);
    dev::mbar_init(k_full, 1);
    for (int i = 0; i < 2; ++i) {
      dev::mbar_init(&qd_full[i], 1);
      dev::mbar_init(&qd_empty[i], 1);
    }
    dev::mbar_init(s_full, 1);
    dev::mbar_init(p_full, 128);
    dev::mbar_init(dq_full, 1);
    dev::mbar_init(s_free, 128);
    dev::mbar_init(v_ready, 128);
    dev::mbar_init(stage_free, 1);
    dev::fence_barrier_init();
  }
  if (warp == 2) dev::tmem_alloc<512>(tmem_slot);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      dev::mbar_arrive_expect_tx(k_full, KT);
#pragma unroll
      for (int c = 0; c < HD / 64; ++c)
        dev::tma_load_2d(sK + c * CH128, &tm_k, k_full, Dl + h * HD + c * 64, row0 + key0);
      for (int n = 0; n < nq; ++n) {
        const int st = n & 1;
        const int qs = key0 + n * BQB;
        dev::mbar_wait(&qd_empty[st], ((n >> 1) & 1) ^ 1);
        dev::mbar_arrive_expect_tx(&qd_full[st], 2 * QB);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          dev::tma_load_2d(sQ + st * QB + c * CH, &tm_q, &qd_full[st], h * HD + c * 64, row0 + qs);
          dev::tma_load_2d(sDO + st * QB + c * CH, &tm_do, &qd_full[st], h * HD + c * 64, row0 + qs);
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t id_s = dev::make_idesc_bf16(128, BQB, 0, 0);    // S^T, dP^T: M keys, N queries, K head dim
    const uint32_t id_k = dev::make_idesc_bf16(128, HD, 0, 1);     // dK: M keys, N head dim, K queries
    const uint32_t id_q = dev::make_idesc_bf16(128, BQB, 1, 1);    // dQ^T: M head dim (half), N queries, K keys
    const uint64_t dK_k = dev::make_sdesc_sw128(dev::smem_u32(sK), 16, 1024);       // K as K-major A
    const uint64_t dK_mn = dev::make_sdesc_sw128(dev::smem_u32(sK), CH128, 1024);   // K^T as MN-major A
    const uint64_t dQ_k = dev::make_sdesc_sw128(dev::smem_u32(sQ), 16, 1024);
    const uint64_t dQ_mn = dev::make_sdesc_sw128(dev::smem_u32(sQ), CH, 1024);
    const uint64_t dDO_k = dev::make_sdesc_sw128(dev::smem_u32(sDO), 16, 1024);
    const uint64_t dDS_mn = dev::make_sdesc_sw128(dev::smem_u32(sDS), CH128, 1024);  // dS^T as MN-major B
    constexpr uint64_t QB16 = QB >> 4;
    dev::mbar_wait(k_full, 0);
    dev::mbar_wait(v_ready, 0);
    dev::tc_fence_after();
    for (int n = 0; n < nq; ++n) {
      const int st = n & 1;
      if (lane == 0) T256(16 * n);
      dev::mbar_wait(&qd_full[st], (n >> 1) & 1);
      if (lane == 0) T256(16 * n + 1);
      if (n > 0) dev::mbar_wait(s_free, (n - 1) & 1);  // dQ^T_{n-1} has left the S^T / dP^T columns
      if (lane == 0) T256(16 * n + 2);
      dev::tc_fence_after();
      const uint64_t q_k = dQ_k + st * QB16, do_k = dDO_k + st * QB16;
      if (dev::elect_one_sync()) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint64_t off = static_cast<uint64_t>((kk >> 2) * (CH >> 4) + (kk & 3) * 2);
          dev::umma_f16_ss(tmem + K_S, dK_k + static_cast<uint64_t>((kk >> 2) * (CH128 >> 4) + (kk & 3) * 2),
                           q_k + off, id_s, kk > 0 ? 1u : 0u);
          dev::umma_f16_ts(tmem + K_DP, tmem + K_V + kk * 8, do_k + off, id_s, kk > 0 ? 1u : 0u);
        }
        dev::umma_commit(s_full);
      }
      __syncwarp();
      dev::mbar_wait(p_full, n & 1);
      if (lane == 0) T256(16 * n + 3);
      dev::tc_fence_after();
      const uint64_t q_mn = dQ_mn + st * QB16;
      if (dev::elect_one_sync()) {
        // dK += dS^T Q_n: dS^T (bf16 pairs) in the first 32 columns of dP^T_n
#pragma unroll
        for (int kk = 0; kk < BQB / 16; ++kk)
          dev::umma_f16_ts(tmem + K_ACC, tmem + K_DP + kk * 8, q_mn + static_cast<uint64_t>(kk * 128), id_k,
                           (n > 0 || kk > 0) ? 1u : 0u);
        // dQ^T_n = K^T dS^T_n: head-dim rows [0, 128) over S^T_n, [128, 256) over dP^T_n (after dK
        // has read dS^T there: MMAs execute in issue order)
#pragma unroll
        for (int half = 0; half < 2; ++half) {
#pragma unroll
          for (int kk = 0; kk < 128 / 16; ++kk)
            dev::umma_f16_ss(tmem + (half ? K_DP : K_S), dK_mn + static_cast<uint64_t>(half * 2 * (CH128 >> 4) + kk * 128),
                             dDS_mn + static_cast<uint64_t>(kk * 128), id_q, kk > 0 ? 1u : 0u);
        }
        dev::umma_commit(dq_full);
        dev::umma_commit(&qd_empty[st]);
      }
      __syncwarp();
    }
  } else if (warp >= 4 && warp < 8) {
    // softmax warpgroup: thread = key row
    const int t = static_cast<int>(warp & 3) * 32 + static_cast<int>(lane);
    const int key = key0 + t;
    const uint32_t lb = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int64_t ld = 3LL * Dl;
    row_to_tmem(qkv + (static_cast<int64_t>(row0) + min(key, T - 1)) * ld + 2 * Dl + h * HD, key < T, tmem + lb + K_V);
    dev::tc_fence_before();
    dev::mbar_arrive(v_ready);
    const float log2e = 1.4426950408889634f;
    const float* lse_bh = lse + static_cast<int64_t>(bh) * T;
    const float* del_bh = delta + static_cast<int64_t>(bh) * T;
    const float2 sl2 = make_float2(scale_log2, scale_log2), sc2 = make_float2(scale, scale);
    for (int n = 0; n < nq; ++n) {
      const int qs = key0 + n * BQB;
      const bool tw = warp == 4 && lane == 0;
      // the block's softmax statistics, one per thread, into shared memory (their load latency
      // overlaps the wait for S^T / dP^T): [-lse log2e (64) | -delta scale (64)]
      {
        const int qq = qs + (t & (BQB - 1));
        const float x = qq < T ? __ldg((t < BQB ? lse_bh : del_bh) + qq) : 0.f;
        sStat[t] = x * (t < BQB ? -log2e : -scale);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (tw) T256(16 * n + 4);
      dev::mbar_wait(s_full, n & 1);
      if (tw) T256(16 * n + 5);
      dev::tc_fence_after();
      uint32_t sv[64], pv[64];
      dev::tmem_ld_32x32b_x32(tmem + lb + K_S, *reinterpret_cast<uint32_t(*)[32]>(sv));
      dev::tmem_ld_32x32b_x32(tmem + lb + K_S + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
      dev::tmem_ld_32x32b_x32(tmem + lb + K_DP, *reinterpret_cast<uint32_t(*)[32]>(pv));
      dev::tmem_ld_32x32b_x32(tmem + lb + K_DP + 32, *reinterpret_cast<uint32_t(*)[32]>(pv + 32));
      dev::tmem_ld_wait();
      const bool masked = qs < key0 + 128 || qs + BQB > T || key0 + 128 > T;
      const float2* nl2 = reinterpret_cast<const float2*>(sStat);
      const float2* nd2 = reinterpret_cast<const float2*>(sStat + BQB);
      auto dsmath = [&](auto kMask) {
#pragma unroll
        for (int e = 0; e < BQB / 2; ++e) {  // P = 2^(s sl - lse log2e), dS = P (dP - delta) scale
          const int qq = qs + 2 * e;
          const float2 a = dev::ffma2(make_float2(__uint_as_float(sv[2 * e]), __uint_as_float(sv[2 * e + 1])), sl2, nl2[e]);
          float p0 = dev::ex2_approx(a.x), p1 = dev::ex2_approx(a.y);
          if constexpr (decltype(kMask)::value) {
            p0 = (qq < T && key < T && qq >= key) ? p0 : 0.f;
            p1 = (qq + 1 < T && key < T && qq + 1 >= key) ? p1 : 0.f;
          }
          const float2 g = dev::ffma2(make_float2(__uint_as_float(pv[2 * e]), __uint_as_float(pv[2 * e + 1])), sc2, nd2[e]);
          const float2 ds = dev::fmul2(make_float2(p0, p1), g);
          sv[e] = dev::pack_bf16x2(ds.x, ds.y);
        }
      };
      if (masked) dsmath(std::true_type{}); else dsmath(std::false_type{});
      // dS^T_n: TMEM (A of dK, over the dP^T columns just read) and shared memory (B of dQ^T).
      // The shared tile was last read by dQ^T_{n-1} (complete before s_full of block n) and then
      // served as dQ_{n-1}'s staging: wait until TMA has read that
      if (n > 0) dev::mbar_wait(stage_free, (n - 1) & 1);
      dev::tmem_st_32x32b_x32(tmem + lb + K_DP, *reinterpret_cast<uint32_t(*)[32]>(sv));
#pragma unroll
      for (int u = 0; u < 8; ++u)
        dev::st_sw128(sDS, 128, t, 0, u, make_uint4(sv[4 * u], sv[4 * u + 1], sv[4 * u + 2], sv[4 * u + 3]));
      dev::tmem_st_wait();
      dev::fence_proxy_async_smem();
      dev::tc_fence_before();
      dev::mbar_arrive(p_full);
      if (tw) T256(16 * n + 6);
      asm volatile("bar.sync 1, 128;" ::: "memory");  // every thread has read this block's statistics
    }
    dev::mbar_wait(dq_full, (nq - 1) & 1);
    dev::tc_fence_after();
    acc_row_out(tmem + lb + K_ACC, dqkv + (static_cast<int64_t>(row0) + key) * ld + Dl + h * HD, key < T);
  } else if (warp >= 8) {
    // dQ warpgroup: thread = head-dim row d of a half. Per half, dQ^T_n (64 query columns) is
    // staged as 4 TMA boxes of [64 queries x 32 fp32] (SW128, a warp writes one 128-byte row per
    // query: conflict-free) and added into the fp32 dQ accumulator by TMA reduce-add
    const int d = static_cast<int>(warp & 3) * 32 + static_cast<int>(lane);
    const uint32_t lb = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int wd = d & 31;
    uint8_t* bx = (d >> 5) < 2 ? sDS + (d >> 5) * (BQB * 128) : sDQX + ((d >> 5) - 2) * (BQB * 128);
    const bool leader = warp == 8 && lane == 0;
    for (int n = 0; n < nq; ++n) {
      const int qs = key0 + n * BQB;
      const bool tw = leader;
      if (tw) T256(16 * n + 7);
      dev::mbar_wait(dq_full, n & 1);
      if (tw) T256(16 * n + 8);
      dev::tc_fence_after();
      // both halves into registers, then the S^T / dP^T columns are handed back at once: the
      // next block's S^T / dP^T MMAs run while this block's dQ is staged and reduced
      uint32_t v[2][64];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const uint32_t src = tmem + lb + (half ? K_DP : K_S);
        dev::tmem_ld_32x32b_x32(src, *reinterpret_cast<uint32_t(*)[32]>(v[half]));
        dev::tmem_ld_32x32b_x32(src + 32, *reinterpret_cast<uint32_t(*)[32]>(v[half] + 32));
      }
      dev::tmem_ld_wait();
      dev::tc_fence_before();
      dev::mbar_arrive(s_free);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        if (half == 1) {  // the first half's reduce-adds have read the staging boxes
          if (leader) dev::bulk_wait_read();
          asm volatile("bar.sync 2, 128;" ::: "memory");
        }
#pragma unroll
        for (int q = 0; q < BQB; ++q)
          *reinterpret_cast<uint32_t*>(bx + q * 128 + (((wd >> 2) ^ (q & 7)) << 4) + (wd & 3) * 4) = v[half][q];
        dev::fence_proxy_async_smem();
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (leader) {
#pragma unroll
          for (int bb = 0; bb < 4; ++bb)
            dev::tma_reduce_add_2d(&tm_dq, bb < 2 ? sDS + bb * (BQB * 128) : sDQX + (bb - 2) * (BQB * 128),
                                   h * HD + half * 128 + bb * 32, row0 + qs);
          dev::bulk_commit();
        }
      }
      // the staging (boxes 0-1 are the dS^T tile) has been read: the softmax may write dS^T_{n+1}
      if (leader) {
        dev::bulk_wait_read();
        dev::mbar_arrive(stage_free);
      }
      __syncwarp();
      if (tw) T256(16 * n + 9);
    }
    if (leader) dev::bulk_wait_all();
  }
  dev::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    dev::tc_fence_after();
    dev::tmem_dealloc<512>(tmem);
  }
}

}  // namespace

void attn_delta(const bf16* o, const bf16* dout, float* delta, int T, int Hl, int hd, int64_t M, cudaStream_t s);
void attn_dq_to_bf16(const float* dq, bf16* dqkv, int64_t M, int Dl, cudaStream_t s);

bool attention_hd256_bwd(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, bf16* dqkv,
                         float* scratch, int B, int T, int Hl, cudaStream_t s, bool delta_ready) {
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(attn_bwd_hd256_dv, cudaFuncAttributeMaxDynamicSharedMemorySize, DvLay::BYTES) !=
            cudaSuccess ||
        cudaFuncSetAttribute(attn_bwd_hd256_dkq, cudaFuncAttributeMaxDynamicSharedMemorySize, DkLay::BYTES) !=
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
  if (!delta_ready) attn_delta(o, dout, delta, T, Hl, HD, M, s);
  const CUtensorMap tm_q = make_tmap_bf16_2d(qkv, 3ull * Dl, static_cast<uint64_t>(M), 3ull * Dl, 64, BQB);
  const CUtensorMap tm_k = make_tmap_bf16_2d(qkv, 3ull * Dl, static_cast<uint64_t>(M), 3ull * Dl, 64, 128);
  const CUtensorMap tm_do = make_tmap_bf16_2d(dout, static_cast<uint64_t>(Dl), static_cast<uint64_t>(M),
                                              static_cast<uint64_t>(Dl), 64, BQB);
  const int nkb = (T + 127) / 128;
  const double scale = 1.0 / std::sqrt(static_cast<double>(HD));
  const float sl = static_cast<float>(scale * 1.4426950408889634);
  // phase traces (SW_ATTN_TRACE_HD256=1 reads them): the dK/dQ pass, or with SW_ATTN_TRACE_DV=1
  // the dV pass (tools/attn256_trace.py, tools/attn256_dv_trace.py)
  static const int trace_cta0 = [] {
    const char* e = std::getenv("SW_ATTN_TRACE_CTA");
    return e != nullptr ? std::atoi(e) : -1;
  }();
  static const bool trace_dv = [] {
    const char* e = std::getenv("SW_ATTN_TRACE_DV");
    return e != nullptr && e[0] == '1';
  }();
  attn_bwd_hd256_dv<<<nkb * B * Hl, 256, DvLay::BYTES, s>>>(tm_q, tm_do, qkv, lse, dqkv, T, Hl, sl, B * Hl,
                                                           trace_dv ? trace_cta0 : -1);
  const int trace_cta = trace_dv ? -1 : trace_cta0;
  const CUtensorMap tm_dq = make_tmap_f32_2d(dq, static_cast<uint64_t>(Dl), static_cast<uint64_t>(M),
                                             static_cast<uint64_t>(Dl), 32, BQB);
  attn_bwd_hd256_dkq<<<nkb * B * Hl, 384, DkLay::BYTES, s>>>(tm_k, tm_q, tm_do, tm_dq, qkv, lse, delta, dqkv, dq, T, Hl, sl,
                                                             static_cast<float>(scale), B * Hl, trace_cta);
  attn_dq_to_bf16(dq, dqkv, M, Dl, s);
  return true;
}

void attention_hd256_trace_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_hd256_trace, sizeof(unsigned long long) * 4096);
}

bool attention_hd256_fwd(const bf16* qkv, bf16* o, float* lse, int B, int T, int Hl, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(attn_fwd_hd256, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdLay::BYTES) !=
        cudaSuccess) {
      return false;
    }
    configured = true;
  }
  const int Dl = Hl * HD;
  const CUtensorMap tm = make_tmap_bf16_2d(qkv, 3ull * Dl, static_cast<uint64_t>(B) * T, 3ull * Dl, 64, BK);
  const int nqb = (T + BQ - 1) / BQ;
  const double scale = 1.0 / std::sqrt(static_cast<double>(HD));
  attn_fwd_hd256<<<nqb * B * Hl, 256, FwdLay::BYTES, s>>>(tm, qkv, o, lse, T, Hl,
                                                         static_cast<float>(scale * 1.4426950408889634),
                                                         static_cast<float>(scale), B * Hl);
  return true;
}

}  // namespace k
}  // namespace sw
