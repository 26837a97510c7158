// Kernels of the T5 encoder-decoder extension (BASELINE cfg4).
//
// Attention here is the general form of the SDPA composite (graph.hpp:650-661): separate q and
// k/v sources (cross-attention reads k/v from the encoder output), Tq != Tk, an optional
// additive relative-position bias [Hl, Tq, Tk] (T5: embedding_lookup of the bucket ids into
// rel_bias [buckets, H], head-sliced per rank as spmd.hpp:398-401 does for a replicated operand
// broadcast against head-split scores), optional causal mask, and T5's unit score scale. One
// warp per query row, fp32 online softmax; the backward recomputes the probabilities from the
// saved log-sum-exp, accumulates dK / dV with fp32 atomics and, when a bias is present, its
// gradient dS summed over the batch (the VJP of the broadcast add).
#include <cmath>

#include "kernels.h"
#include "sm100.cuh"

namespace sw {
namespace k {

namespace {

constexpr int kMaxPerLane = 8;  // head dim <= 256

__device__ __forceinline__ float warp_sum32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void t5_attn_fwd_kernel(T5AttnArgs a) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (i >= a.Tq) return;
  const int bh = blockIdx.y, b = bh / a.Hl, h = bh % a.Hl;
  const bf16* qr = a.q + (static_cast<int64_t>(b) * a.Tq + i) * a.ldq + h * a.dk;
  float q[kMaxPerLane], acc[kMaxPerLane];
#pragma unroll
  for (int u = 0; u < kMaxPerLane; ++u) {
    const int c = lane + 32 * u;
    q[u] = c < a.dk ? __bfloat162float(qr[c]) : 0.f;
    acc[u] = 0.f;
  }
  const float* brow = a.bias ? a.bias + (static_cast<int64_t>(h) * a.Tq + i) * a.Tk : nullptr;
  const int jend = a.causal ? (i + 1 < a.Tk ? i + 1 : a.Tk) : a.Tk;
  float m = -INFINITY, l = 0.f;
  for (int j = 0; j < jend; ++j) {
    const int64_t rj = static_cast<int64_t>(b) * a.Tk + j;
    const bf16* kr = a.k + rj * a.ldk + h * a.dk;
    const bf16* vr = a.v + rj * a.ldv + h * a.dk;
    float p = 0.f;
#pragma unroll
    for (int u = 0; u < kMaxPerLane; ++u) {
      const int c = lane + 32 * u;
      if (c < a.dk) p += q[u] * __bfloat162float(kr[c]);
    }
    float sc = warp_sum32(p) * a.scale;
    if (brow) sc += brow[j];
    const float mn = fmaxf(m, sc);
    const float corr = __expf(m - mn);
    const float e = __expf(sc - mn);
    l = l * corr + e;
#pragma unroll
    for (int u = 0; u < kMaxPerLane; ++u) {
      const int c = lane + 32 * u;
      if (c < a.dk) acc[u] = acc[u] * corr + e * __bfloat162float(vr[c]);
    }
    m = mn;
  }
  bf16* orow = a.o + (static_cast<int64_t>(b) * a.Tq + i) * a.ldo + h * a.dk;
  const float inv = 1.f / l;
#pragma unroll
  for (int u = 0; u < kMaxPerLane; ++u) {
    const int c = lane + 32 * u;
    if (c < a.dk) orow[c] = __float2bfloat16(acc[u] * inv);
  }
  if (lane == 0) a.lse[static_cast<int64_t>(bh) * a.Tq + i] = m + logf(l);
}

// delta[b,h,i] = sum_c dO[i,c] * O[i,c]
__global__ void t5_attn_delta_kernel(T5AttnArgs a, const bf16* __restrict__ dout, int64_t ldd,
                                     float* __restrict__ delta) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (i >= a.Tq) return;
  const int bh = blockIdx.y, b = bh / a.Hl, h = bh % a.Hl;
  const int64_t row = static_cast<int64_t>(b) * a.Tq + i;
  float s = 0.f;
  for (int c = lane; c < a.dk; c += 32)
    s += __bfloat162float(a.o[row * a.ldo + h * a.dk + c]) * __bfloat162float(dout[row * ldd + h * a.dk + c]);
  s = warp_sum32(s);
  if (lane == 0) delta[static_cast<int64_t>(bh) * a.Tq + i] = s;
}

__global__ void t5_attn_bwd_kernel(T5AttnArgs a, const bf16* __restrict__ dout, int64_t ldd,
                                   const float* __restrict__ delta, bf16* __restrict__ dq, int64_t lddq,
                                   float* __restrict__ dkv, float* __restrict__ dbias) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (i >= a.Tq) return;
  const int bh = blockIdx.y, b = bh / a.Hl, h = bh % a.Hl;
  const int Dl = a.Hl * a.dk;
  const int64_t row_i = static_cast<int64_t>(b) * a.Tq + i;
  float q[kMaxPerLane], dO[kMaxPerLane], g[kMaxPerLane];
#pragma unroll
  for (int u = 0; u < kMaxPerLane; ++u) {
    const int c = lane + 32 * u;
    q[u] = c < a.dk ? __bfloat162float(a.q[row_i * a.ldq + h * a.dk + c]) : 0.f;
    dO[u] = c < a.dk ? __bfloat162float(dout[row_i * ldd + h * a.dk + c]) : 0.f;
    g[u] = 0.f;
  }
  const float L = a.lse[static_cast<int64_t>(bh) * a.Tq + i];
  const float D = delta[static_cast<int64_t>(bh) * a.Tq + i];
  const float* brow = a.bias ? a.bias + (static_cast<int64_t>(h) * a.Tq + i) * a.Tk : nullptr;
  float* dbrow = dbias ? dbias + (static_cast<int64_t>(h) * a.Tq + i) * a.Tk : nullptr;
  const int jend = a.causal ? (i + 1 < a.Tk ? i + 1 : a.Tk) : a.Tk;
  for (int j = 0; j < jend; ++j) {
    const int64_t rj = static_cast<int64_t>(b) * a.Tk + j;
    const bf16* kr = a.k + rj * a.ldk + h * a.dk;
    const bf16* vr = a.v + rj * a.ldv + h * a.dk;
    float s = 0.f, dp = 0.f;
#pragma unroll
    for (int u = 0; u < kMaxPerLane; ++u) {
      const int c = lane + 32 * u;
      if (c < a.dk) {
        s += q[u] * __bfloat162float(kr[c]);
        dp += dO[u] * __bfloat162float(vr[c]);
      }
    }
    s = warp_sum32(s) * a.scale;
    if (brow) s += brow[j];
    dp = warp_sum32(dp);
    const float p = __expf(s - L);
    const float gs = p * (dp - D);  // d loss / d score (also the bias gradient)
    if (dbrow && lane == 0) atomicAdd(dbrow + j, gs);
    const float ds = gs * a.scale;
    float* dk = dkv + rj * (2LL * Dl) + h * a.dk;
    float* dv = dk + Dl;
#pragma unroll
    for (int u = 0; u < kMaxPerLane; ++u) {
      const int c = lane + 32 * u;
      if (c < a.dk) {
        g[u] += ds * __bfloat162float(kr[c]);
        atomicAdd(dk + c, ds * q[u]);
        atomicAdd(dv + c, p * dO[u]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kMaxPerLane; ++u) {
    const int c = lane + 32 * u;
    if (c < a.dk) dq[row_i * lddq + h * a.dk + c] = __float2bfloat16(g[u]);
  }
}

__global__ void t5_dkv_out_kernel(const float* __restrict__ dkv, bf16* __restrict__ dk, int64_t lddk,
                                  bf16* __restrict__ dv, int64_t lddv, int64_t M, int Dl) {
  const int64_t n = M * 2LL * Dl;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / (2LL * Dl), c = e - r * (2LL * Dl);
    if (c < Dl)
      dk[r * lddk + c] = __float2bfloat16(dkv[e]);
    else
      dv[r * lddv + c - Dl] = __float2bfloat16(dkv[e]);
  }
}

// bias[h, i, j] = table[ids[i, j], h0 + h]   (table [buckets, H] row-major)
__global__ void t5_bias_build_kernel(const float* __restrict__ table, const int32_t* __restrict__ ids, int H,
                                     int h0, int Hl, int64_t TT, float* __restrict__ bias) {
  const int64_t n = static_cast<int64_t>(Hl) * TT;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t h = e / TT, ij = e - h * TT;
    bias[e] = table[static_cast<int64_t>(ids[ij]) * H + h0 + h];
  }
}

// table_grad[bucket, h0 + h] += sum_{(i,j): ids[i,j] == bucket} dbias[h, i, j]: one CTA per
// (head, slice of positions), bucket sums in shared memory, one global atomic per bucket.
__global__ void t5_bias_grad_kernel(const float* __restrict__ dbias, const int32_t* __restrict__ ids, int H,
                                    int h0, int64_t TT, int nb, float* __restrict__ table_grad) {
  extern __shared__ float acc[];
  for (int t = threadIdx.x; t < nb; t += blockDim.x) acc[t] = 0.f;
  __syncthreads();
  const int h = blockIdx.y;
  const float* src = dbias + static_cast<int64_t>(h) * TT;
  for (int64_t ij = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; ij < TT;
       ij += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    atomicAdd(&acc[ids[ij]], src[ij]);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nb; t += blockDim.x) atomicAdd(table_grad + static_cast<int64_t>(t) * H + h0 + h, acc[t]);
}

__global__ void t5_lut_build_kernel(const float* __restrict__ table, const int32_t* __restrict__ bucket, int H,
                                    int h0, int Hl, int T, float* __restrict__ lut) {
  const int64_t W = 2LL * T + 128, n = static_cast<int64_t>(Hl) * W;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t h = e / W, i = e - h * W;
    lut[e] = i < 2LL * T - 1 ? table[static_cast<int64_t>(bucket[i]) * H + h0 + h] : 0.f;
  }
}

__global__ void t5_lut_grad_kernel(const float* __restrict__ dlut, const int32_t* __restrict__ bucket, int H,
                                   int h0, int T, float* __restrict__ table_grad) {
  const int h = blockIdx.y;
  const float* src = dlut + static_cast<int64_t>(h) * (2LL * T + 128);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * T - 1; i += gridDim.x * blockDim.x) {
    const float g = src[i];
    if (g != 0.f) atomicAdd(table_grad + static_cast<int64_t>(bucket[i]) * H + h0 + h, g);
  }
}

unsigned blocks_for(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return static_cast<unsigned>(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

}  // namespace

void t5_attention_fwd(const T5AttnArgs& a, int B, cudaStream_t s) {
  dim3 grid((a.Tq + 3) / 4, B * a.Hl);
  t5_attn_fwd_kernel<<<grid, 128, 0, s>>>(a);
}

void t5_attention_bwd(const T5AttnArgs& a, int B, const bf16* dout, int64_t ldd, bf16* dq, int64_t lddq, bf16* dk,
                      int64_t lddk, bf16* dv, int64_t lddv, float* scratch, float* dbias, cudaStream_t s) {
  const int Dl = a.Hl * a.dk;
  const int64_t Mk = static_cast<int64_t>(B) * a.Tk;
  float* delta = scratch;
  float* dkv = scratch + ((static_cast<int64_t>(B) * a.Hl * a.Tq + 63) / 64) * 64;
  cudaMemsetAsync(dkv, 0, sizeof(float) * Mk * 2 * Dl, s);
  dim3 grid((a.Tq + 3) / 4, B * a.Hl);
  t5_attn_delta_kernel<<<grid, 128, 0, s>>>(a, dout, ldd, delta);
  t5_attn_bwd_kernel<<<grid, 128, 0, s>>>(a, dout, ldd, delta, dq, lddq, dkv, dbias);
  t5_dkv_out_kernel<<<blocks_for(Mk * 2 * Dl), 256, 0, s>>>(dkv, dk, lddk, dv, lddv, Mk, Dl);
}

int64_t t5_attention_scratch(int B, int Hl, int Tq, int Tk, int dk) {
  return ((static_cast<int64_t>(B) * Hl * Tq + 63) / 64) * 64 + static_cast<int64_t>(B) * Tk * 2 * Hl * dk;
}

void t5_bias_build(const float* table, const int32_t* ids, int H, int h0, int Hl, int64_t TT, float* bias,
                   cudaStream_t s) {
  t5_bias_build_kernel<<<blocks_for(static_cast<int64_t>(Hl) * TT), 256, 0, s>>>(table, ids, H, h0, Hl, TT, bias);
}

void t5_bias_grad(const float* dbias, const int32_t* ids, int H, int h0, int Hl, int64_t TT, int nb,
                  float* table_grad, cudaStream_t s) {
  const int64_t per = 256 * 16;
  dim3 grid(static_cast<unsigned>((TT + per - 1) / per), Hl);
  t5_bias_grad_kernel<<<grid, 256, nb * sizeof(float), s>>>(dbias, ids, H, h0, TT, nb, table_grad);
}

void t5_lut_build(const float* table, const int32_t* bucket, int H, int h0, int Hl, int T, float* lut, cudaStream_t s) {
  t5_lut_build_kernel<<<blocks_for(static_cast<int64_t>(Hl) * (2LL * T + 128)), 256, 0, s>>>(table, bucket, H, h0, Hl, T,
                                                                                          lut);
}

void t5_lut_grad(const float* dlut, const int32_t* bucket, int H, int h0, int Hl, int T, float* table_grad,
                 cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((2 * T + 255) / 256), Hl);
  t5_lut_grad_kernel<<<grid, 256, 0, s>>>(dlut, bucket, H, h0, T, table_grad);
}


}  // namespace k
}  // namespace sw
