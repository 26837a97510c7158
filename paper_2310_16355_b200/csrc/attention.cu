// Head-sharded causal attention (graph.hpp:650-661 with the additive -1e9 causal mask of
// model.hpp:100-106; masked probabilities are exactly zero, so masked keys are skipped).
//
// Layout: qkv [B*T, 3*Dl] bf16 with q | k | v blocks, head h at column h*hd of each block;
// o [B*T, Dl] bf16 (feeds the row-parallel output projection directly); lse [B, Hl, T] fp32.
//
// This file holds the generic (any head_dim <= 256) warp-per-query kernels; the tensor-core
// kernels for head_dim 64/128 live in attention_mma.cu and are preferred when they apply.
#include <cmath>

#include "kernels.h"
#include "sm100.cuh"

namespace sw {
namespace k {

bool attention_mma_fwd(const bf16* qkv, bf16* o, float* lse, int B, int T, int Hl, int hd,
                       cudaStream_t s);
bool attention_mma_bwd(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout,
                       bf16* dqkv, float* scratch, int B, int T, int Hl, int hd, cudaStream_t s,
                       bool delta_ready, float* colsum, bool* colsum_done);
bool attention_mma_fwd_ex(const bf16* qkv, bf16* o, float* lse, int B, int T, int Hl, int hd, int causal,
                          const float* lut, float scale, cudaStream_t s);
bool attention_mma_bwd_ex(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, bf16* dqkv,
                          float* scratch, int B, int T, int Hl, int hd, int causal, const float* lut, float* dlut,
                          float scale, cudaStream_t s);
bool attention_mma_fwd_cross(const bf16* q, int64_t ldq, const bf16* kv, int64_t ldkv, int voff, bf16* o, float* lse,
                             int B, int Tq, int Tk, int Hl, int hd, float scale, cudaStream_t s);
bool attention_mma_bwd_cross(const bf16* q, int64_t ldq, const bf16* kv, int64_t ldkv, int voff, const bf16* o,
                             const float* lse, const bf16* dout, bf16* dq, int64_t ld_dq, bf16* dkv, int64_t ld_dkv,
                             float* scratch, int B, int Tq, int Tk, int Hl, int hd, float scale, cudaStream_t s);

namespace {

constexpr int kMaxPerLane = 8;  // head_dim <= 256

__device__ __forceinline__ float wsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void attn_fwd_generic(const bf16* __restrict__ qkv, bf16* __restrict__ o,
                                 float* __restrict__ lse, int T, int Hl, int hd, float scale) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (i >= T) return;
  const int bh = blockIdx.y, b = bh / Hl, h = bh % Hl;
  const int Dl = Hl * hd;
  const int64_t ld = 3LL * Dl;
  const bf16* qr = qkv + (static_cast<int64_t>(b) * T + i) * ld + h * hd;
  float q[kMaxPerLane], acc[kMaxPerLane];
#pragma unroll
  for (int u = 0; u < kMaxPerLane; ++u) {
    const int c = lane + 32 * u;
    q[u] = c < hd ? __bfloat162float(qr[c]) : 0.f;
    acc[u] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int j = 0; j <= i; ++j) {
    const bf16* kr = qkv + (static_cast<int64_t>(b) * T + j) * ld + Dl + h * hd;
    float p = 0.f;
#pragma unroll
    for (int u = 0; u < kMaxPerLane; ++u) {
      const int c = lane + 32 * u;
      if (c < hd) p += q[u] * __bfloat162float(kr[c]);
    }
    const float sc = wsum(p) * scale;
    const float mn = fmaxf(m, sc);
    const float corr = __expf(m - mn);
    const float e = __expf(sc - mn);
    l = l * corr + e;
    const bf16* vr = kr + Dl;
#pragma unroll
    for (int u = 0; u < kMaxPerLane; ++u) {
      const int c = lane + 32 * u;
      if (c < hd) acc[u] = acc[u] * corr + e * __bfloat162float(vr[c]);
    }
    m = mn;
  }
  bf16* orow = o + (static_cast<int64_t>(b) * T + i) * Dl + h * hd;
  const float inv = 1.f / l;
#pragma unroll
  for (int u = 0; u < kMaxPerLane; ++u) {
    const int c = lane + 32 * u;
    if (c < hd) orow[c] = __float2bfloat16(acc[u] * inv);
  }
  if (lane == 0) lse[(static_cast<int64_t>(bh)) * T + i] = m + logf(l);
}

// delta[b,h,i] = sum_c dO[i,c] * O[i,c]
__global__ void attn_bwd_delta(const bf16* __restrict__ o, const bf16* __restrict__ dout,
                               float* __restrict__ delta, int T, int Hl, int hd) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (i >= T) return;
  const int bh = blockIdx.y, b = bh / Hl, h = bh % Hl;
  const int64_t off = (static_cast<int64_t>(b) * T + i) * (Hl * hd) + h * hd;
  float s = 0.f;
  for (int c = lane; c < hd; c += 32) s += __bfloat162float(o[off + c]) * __bfloat162float(dout[off + c]);
  s = wsum(s);
  if (lane == 0) delta[static_cast<int64_t>(bh) * T + i] = s;
}

// One warp per query i: dQ_i directly; dK_j, dV_j accumulated with fp32 atomics into dkv
// [B*T, 2*Dl] (k block then v block).
__global__ void attn_bwd_generic(const bf16* __restrict__ qkv, const float* __restrict__ lse,
                                 const float* __restrict__ delta, const bf16* __restrict__ dout,
                                 bf16* __restrict__ dqkv, float* __restrict__ dkv, int T, int Hl,
                                 int hd, float scale) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (i >= T) return;
  const int bh = blockIdx.y, b = bh / Hl, h = bh % Hl;
  const int Dl = Hl * hd;
  const int64_t ld = 3LL * Dl;
  const int64_t row_i = static_cast<int64_t>(b) * T + i;
  float q[kMaxPerLane], dO[kMaxPerLane], dq[kMaxPerLane];
#pragma unroll
  for (int u = 0; u < kMaxPerLane; ++u) {
    const int c = lane + 32 * u;
    q[u] = c < hd ? __bfloat162float(qkv[row_i * ld + h * hd + c]) : 0.f;
    dO[u] = c < hd ? __bfloat162float(dout[row_i * Dl + h * hd + c]) : 0.f;
    dq[u] = 0.f;
  }
  const float L = lse[static_cast<int64_t>(bh) * T + i];
  const float D = delta[static_cast<int64_t>(bh) * T + i];
  for (int j = 0; j <= i; ++j) {
    const int64_t row_j = static_cast<int64_t>(b) * T + j;
    const bf16* kr = qkv + row_j * ld + Dl + h * hd;
    const bf16* vr = kr + Dl;
    float s = 0.f, dp = 0.f;
#pragma unroll
    for (int u = 0; u < kMaxPerLane; ++u) {
      const int c = lane + 32 * u;
      if (c < hd) {
        s += q[u] * __bfloat162float(kr[c]);
        dp += dO[u] * __bfloat162float(vr[c]);
      }
    }
    s = wsum(s) * scale;
    dp = wsum(dp);
    const float p = __expf(s - L);
    const float ds = p * (dp - D) * scale;
    float* dk = dkv + row_j * (2LL * Dl) + h * hd;
    float* dv = dk + Dl;
#pragma unroll
    for (int u = 0; u < kMaxPerLane; ++u) {
      const int c = lane + 32 * u;
      if (c < hd) {
        dq[u] += ds * __bfloat162float(kr[c]);
        atomicAdd(dk + c, ds * q[u]);
        atomicAdd(dv + c, p * dO[u]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kMaxPerLane; ++u) {
    const int c = lane + 32 * u;
    if (c < hd) dqkv[row_i * ld + h * hd + c] = __float2bfloat16(dq[u]);
  }
}

__global__ void dkv_to_bf16(const float* __restrict__ dkv, bf16* __restrict__ dqkv, int64_t M, int Dl) {
  const int64_t n = M * 2LL * Dl;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / (2LL * Dl), c = e - r * (2LL * Dl);
    dqkv[r * 3LL * Dl + Dl + c] = __float2bfloat16(dkv[e]);
  }
}

}  // namespace

void attention_fwd(const bf16* qkv, bf16* o, float* lse, int B, int T, int Hl, int hd,
                   cudaStream_t s) {
  if (attention_mma_fwd(qkv, o, lse, B, T, Hl, hd, s)) return;
  dim3 grid((T + 3) / 4, B * Hl);
  attn_fwd_generic<<<grid, 128, 0, s>>>(qkv, o, lse, T, Hl, hd,
                                        static_cast<float>(1.0 / std::sqrt(static_cast<double>(hd))));
}

void attention_bwd(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, bf16* dqkv,
                   float* scratch, int B, int T, int Hl, int hd, cudaStream_t s, bool delta_ready, float* colsum,
                   bool* colsum_done) {
  if (colsum_done != nullptr) *colsum_done = false;
  if (attention_mma_bwd(qkv, o, lse, dout, dqkv, scratch, B, T, Hl, hd, s, delta_ready, colsum, colsum_done)) return;
  const int64_t M = static_cast<int64_t>(B) * T;
  const int Dl = Hl * hd;
  float* delta = scratch;
  float* dkv = scratch + static_cast<int64_t>(B) * Hl * T;
  cudaMemsetAsync(dkv, 0, sizeof(float) * M * 2 * Dl, s);
  dim3 grid((T + 3) / 4, B * Hl);
  attn_bwd_delta<<<grid, 128, 0, s>>>(o, dout, delta, T, Hl, hd);
  attn_bwd_generic<<<grid, 128, 0, s>>>(qkv, lse, delta, dout, dqkv, dkv, T, Hl, hd,
                                        static_cast<float>(1.0 / std::sqrt(static_cast<double>(hd))));
  dkv_to_bf16<<<1184, 256, 0, s>>>(dkv, dqkv, M, Dl);
}

bool attention_fwd_ex(const bf16* qkv, bf16* o, float* lse, int B, int T, int Hl, int hd, int causal,
                      const float* lut, float scale, cudaStream_t s) {
  return attention_mma_fwd_ex(qkv, o, lse, B, T, Hl, hd, causal, lut, scale, s);
}

bool attention_bwd_ex(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, bf16* dqkv,
                      float* scratch, int B, int T, int Hl, int hd, int causal, const float* lut, float* dlut,
                      float scale, cudaStream_t s) {
  return attention_mma_bwd_ex(qkv, o, lse, dout, dqkv, scratch, B, T, Hl, hd, causal, lut, dlut, scale, s);
}

bool attention_fwd_cross(const bf16* q, int64_t ldq, const bf16* kv, int64_t ldkv, int voff, bf16* o, float* lse,
                         int B, int Tq, int Tk, int Hl, int hd, float scale, cudaStream_t s) {
  return attention_mma_fwd_cross(q, ldq, kv, ldkv, voff, o, lse, B, Tq, Tk, Hl, hd, scale, s);
}

bool attention_bwd_cross(const bf16* q, int64_t ldq, const bf16* kv, int64_t ldkv, int voff, const bf16* o,
                         const float* lse, const bf16* dout, bf16* dq, int64_t ld_dq, bf16* dkv, int64_t ld_dkv,
                         float* scratch, int B, int Tq, int Tk, int Hl, int hd, float scale, cudaStream_t s) {
  return attention_mma_bwd_cross(q, ldq, kv, ldkv, voff, o, lse, dout, dq, ld_dq, dkv, ld_dkv, scratch, B, Tq, Tk, Hl,
                                 hd, scale, s);
}

}  // namespace k
}  // namespace sw
