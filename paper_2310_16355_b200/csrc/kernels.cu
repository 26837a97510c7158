#include <cstdlib>
// Non-GEMM kernels of the tensor-parallel step: embeddings, LayerNorm, bias-gradient column
// sums, fused cross entropy, residual adds, AdamW, emulated collectives and device-side
// parameter init. All are HBM-bound; they use 16-byte vector accesses where the row pitch
// allows and grid-stride loops sized to the SM count.
#include <cmath>
#include <stdexcept>
#include <cstdint>

#include "kernels.h"
#include "sm100.cuh"

namespace sw {
namespace k {

namespace {

constexpr int kSMs = 148;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Sum over the block; every thread receives the total. `red` must hold 32 floats.
__device__ __forceinline__ float block_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  float t = lane < nw ? red[lane] : 0.f;
  return warp_sum(t);
}

inline int grid_for(int64_t n, int threads, int per_thread = 1) {
  int64_t g = (n + static_cast<int64_t>(threads) * per_thread - 1) / (static_cast<int64_t>(threads) * per_thread);
  if (g > 8 * kSMs) g = 8 * kSMs;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

// ------------------------------------------------------------------------------------------
// embeddings
// ------------------------------------------------------------------------------------------
__global__ void embed_fwd_kernel(const int32_t* __restrict__ ids, const float* __restrict__ tok,
                                 const float* __restrict__ pos, float* __restrict__ h, int T, int d) {
  const int64_t m = blockIdx.x;
  const int64_t id = ids[m];
  const int t = static_cast<int>(m % T);
  const float* a = tok + id * d;
  const float* b = pos ? pos + static_cast<int64_t>(t) * d : nullptr;  // T5: no position table
  float* o = h + m * d;
  if ((d & 3) == 0) {
    for (int i = threadIdx.x * 4; i < d; i += blockDim.x * 4) {
      float4 x = *reinterpret_cast<const float4*>(a + i);
      float4 y = b ? *reinterpret_cast<const float4*>(b + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(o + i) = make_float4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w);
    }
  } else {
    for (int i = threadIdx.x; i < d; i += blockDim.x) o[i] = a[i] + (b ? b[i] : 0.f);
  }
}

__global__ void embed_bwd_tok_kernel(const int32_t* __restrict__ ids, const float* __restrict__ g,
                                     float* __restrict__ dtok, int d) {
  const int64_t m = blockIdx.x;
  const int64_t id = ids[m];
  for (int i = threadIdx.x; i < d; i += blockDim.x) atomicAdd(dtok + id * d + i, g[m * d + i]);
}

// keys[i] = (token << 16) | position, padded with 0xffffffff, bitonic-sorted by one CTA.
__global__ void __launch_bounds__(1024) sort_token_keys_kernel(const int32_t* __restrict__ ids, int64_t M, int n,
                                                               uint32_t* __restrict__ keys) {
  extern __shared__ uint32_t sk[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    sk[i] = i < M ? (static_cast<uint32_t>(ids[i]) << 16) | static_cast<uint32_t>(i) : 0xffffffffu;
  }
  __syncthreads();
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint32_t a = sk[i], b = sk[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            sk[i] = b;
            sk[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) keys[i] = sk[i];
}

// Each CTA owns the token runs that start in its slice of the sorted keys and sums the run's
// gradient rows in ascending position order; one owner per token row -> plain (non-atomic) +=.
__global__ void embed_accum_sorted_kernel(const uint32_t* __restrict__ keys, int64_t M, const float* __restrict__ g,
                                          float* __restrict__ dtok, int d, int64_t per_cta) {
  const int64_t i0 = blockIdx.x * per_cta;
  const int64_t i1 = i0 + per_cta < M ? i0 + per_cta : M;
  for (int64_t i = i0; i < i1; ++i) {
    const uint32_t tok = keys[i] >> 16;
    if (i > 0 && (keys[i - 1] >> 16) == tok) continue;  // not the start of a run
    int64_t e = i + 1;
    while (e < M && (keys[e] >> 16) == tok) ++e;
    float* dst = dtok + static_cast<int64_t>(tok) * d;
    for (int c = threadIdx.x * 4; c < d; c += blockDim.x * 4) {
      float4 acc = *reinterpret_cast<const float4*>(dst + c);
      for (int64_t r = i; r < e; ++r) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(g + static_cast<int64_t>(keys[r] & 0xffffu) * d + c));
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      *reinterpret_cast<float4*>(dst + c) = acc;
    }
  }
}

__global__ void embed_bwd_pos_kernel(const float* __restrict__ g, float* __restrict__ dpos, int B,
                                     int T, int d, int accumulate) {
  const int t = blockIdx.x;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float s = 0.f;
    for (int b = 0; b < B; ++b) s += g[(static_cast<int64_t>(b) * T + t) * d + i];
    float* o = dpos + static_cast<int64_t>(t) * d + i;
    *o = accumulate ? *o + s : s;
  }
}

// ------------------------------------------------------------------------------------------
// LayerNorm
// ------------------------------------------------------------------------------------------
template <int THREADS, int V4>
__global__ void __launch_bounds__(THREADS) ln_fwd_kernel(const float* __restrict__ x,
                                                         const float* __restrict__ scale,
                                                         const float* __restrict__ bias,
                                                         bf16* __restrict__ y, float* __restrict__ mean_out,
                                                         float* __restrict__ rstd_out, int d, float eps,
                                                         int rms) {
  __shared__ float red[32];
  const int64_t row = blockIdx.x;
  const float* xr = x + row * d;
  float4 v[V4];
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < V4; ++j) {
    const int c = (threadIdx.x + j * THREADS) * 4;
    v[j] = c < d ? *reinterpret_cast<const float4*>(xr + c) : make_float4(0, 0, 0, 0);
    s += v[j].x + v[j].y + v[j].z + v[j].w;
  }
  // RMSNorm (extension): no centring, no bias -- xhat = x / sqrt(mean(x^2) + eps)
  const float mean = rms ? 0.f : block_sum(s, red) / d;
  float q = 0.f;
#pragma unroll
  for (int j = 0; j < V4; ++j) {
    const int c = (threadIdx.x + j * THREADS) * 4;
    if (c < d) {
      const float a = v[j].x - mean, b = v[j].y - mean, e = v[j].z - mean, f = v[j].w - mean;
      q += a * a + b * b + e * e + f * f;
    }
  }
  const float var = block_sum(q, red) / d;
  const float rstd = 1.0f / sqrtf(var + eps);
  bf16* yr = y + row * d;
#pragma unroll
  for (int j = 0; j < V4; ++j) {
    const int c = (threadIdx.x + j * THREADS) * 4;
    if (c < d) {
      const float4 sc = *reinterpret_cast<const float4*>(scale + c);
      const float4 bi = rms ? make_float4(0.f, 0.f, 0.f, 0.f) : *reinterpret_cast<const float4*>(bias + c);
      uint2 w;
      w.x = dev::pack_bf16x2((v[j].x - mean) * rstd * sc.x + bi.x, (v[j].y - mean) * rstd * sc.y + bi.y);
      w.y = dev::pack_bf16x2((v[j].z - mean) * rstd * sc.z + bi.z, (v[j].w - mean) * rstd * sc.w + bi.w);
      *reinterpret_cast<uint2*>(yr + c) = w;
    }
  }
  if (threadIdx.x == 0) {
    if (mean_out != nullptr) mean_out[row] = mean;
    rstd_out[row] = rstd;
  }
}

// Any d (scalar path).
__global__ void ln_fwd_generic_kernel(const float* __restrict__ x, const float* __restrict__ scale,
                                      const float* __restrict__ bias, bf16* __restrict__ y,
                                      float* __restrict__ mean_out, float* __restrict__ rstd_out,
                                      int d, float eps, int rms) {
  __shared__ float red[32];
  const int64_t row = blockIdx.x;
  const float* xr = x + row * d;
  float s = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) s += xr[i];
  const float mean = rms ? 0.f : block_sum(s, red) / d;
  float q = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float a = xr[i] - mean;
    q += a * a;
  }
  const float var = block_sum(q, red) / d;
  const float rstd = 1.0f / sqrtf(var + eps);
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    y[row * d + i] = __float2bfloat16((xr[i] - mean) * rstd * scale[i] + (rms ? 0.f : bias[i]));
  }
  if (threadIdx.x == 0) {
    if (mean_out != nullptr) mean_out[row] = mean;
    rstd_out[row] = rstd;
  }
}

// dy loaders: the residual-stream gradient arrives as fp32, or as bf16 after a bf16 all-reduce
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float4 ldg4(const bf16* p) {
  const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
  const float2 a = dev::unpack_bf16x2(u.x), b = dev::unpack_bf16x2(u.y);
  return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ float ld1(const float* p) { return *p; }
__device__ __forceinline__ float ld1(const bf16* p) { return __bfloat162float(*p); }

// One CTA walks rows r = blockIdx.x, +gridDim.x, ...; each thread owns fixed columns and
// accumulates dscale / dbias partials in registers, flushed with one atomic per column.
// Two passes per row: pass 1 reduces sum(g) and sum(g*xhat) while accumulating the parameter
// partials; pass 2 re-reads x / dy (L1/L2 hits) to emit dx. Keeping nothing row-sized in
// registers lets four CTAs share an SM, which is what the HBM stream needs.
template <int THREADS, int V4, typename DY>
__global__ void __launch_bounds__(THREADS, (THREADS <= 256 ? 4 : 2)) ln_bwd_kernel(
    const float* __restrict__ x, const float* __restrict__ mean, const float* __restrict__ rstd,
    const float* __restrict__ scale, const DY* __restrict__ dy, float* __restrict__ g_io,
    bf16* __restrict__ g_bf16, float* __restrict__ dscale, float* __restrict__ dbias, int64_t M,
    int d, int accumulate, float* __restrict__ partials, int rms) {
  __shared__ float red[32];
  float4 ds[V4], db[V4];
#pragma unroll
  for (int j = 0; j < V4; ++j) ds[j] = db[j] = make_float4(0, 0, 0, 0);
  for (int64_t row = blockIdx.x; row < M; row += gridDim.x) {
    const float mu = mean ? mean[row] : 0.f, rs = rstd[row];
    const float* xr = x + row * d;
    const DY* dr = dy + row * d;
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < V4; ++j) {
      const int c = (threadIdx.x + j * THREADS) * 4;
      if (c < d) {
        const float4 xv = __ldg(reinterpret_cast<const float4*>(xr + c));
        const float4 dv = ldg4(dr + c);
        const float4 sc = __ldg(reinterpret_cast<const float4*>(scale + c));
        const float4 xh = make_float4((xv.x - mu) * rs, (xv.y - mu) * rs, (xv.z - mu) * rs, (xv.w - mu) * rs);
        ds[j].x += dv.x * xh.x; ds[j].y += dv.y * xh.y; ds[j].z += dv.z * xh.z; ds[j].w += dv.w * xh.w;
        db[j].x += dv.x; db[j].y += dv.y; db[j].z += dv.z; db[j].w += dv.w;
        const float gx = dv.x * sc.x, gy = dv.y * sc.y, gz = dv.z * sc.z, gw = dv.w * sc.w;
        s1 += gx + gy + gz + gw;
        s2 += gx * xh.x + gy * xh.y + gz * xh.z + gw * xh.w;
      }
    }
    const float gm = rms ? 0.f : block_sum(s1, red) / d;  // RMSNorm: no mean term
    const float gxm = block_sum(s2, red) / d;
#pragma unroll
    for (int j = 0; j < V4; ++j) {
      const int c = (threadIdx.x + j * THREADS) * 4;
      if (c < d) {
        const float4 xv = __ldg(reinterpret_cast<const float4*>(xr + c));
        const float4 dv = ldg4(dr + c);
        const float4 sc = __ldg(reinterpret_cast<const float4*>(scale + c));
        float4 dx;
        dx.x = rs * (dv.x * sc.x - gm - (xv.x - mu) * rs * gxm);
        dx.y = rs * (dv.y * sc.y - gm - (xv.y - mu) * rs * gxm);
        dx.z = rs * (dv.z * sc.z - gm - (xv.z - mu) * rs * gxm);
        dx.w = rs * (dv.w * sc.w - gm - (xv.w - mu) * rs * gxm);
        float* gp = g_io + row * d + c;
        if (accumulate) {
          const float4 o = *reinterpret_cast<const float4*>(gp);
          dx.x += o.x; dx.y += o.y; dx.z += o.z; dx.w += o.w;
        }
        *reinterpret_cast<float4*>(gp) = dx;
        uint2 w;
        w.x = dev::pack_bf16x2(dx.x, dx.y);
        w.y = dev::pack_bf16x2(dx.z, dx.w);
        *reinterpret_cast<uint2*>(g_bf16 + row * d + c) = w;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < V4; ++j) {
    const int c = (threadIdx.x + j * THREADS) * 4;
    if (c < d) {
      if (partials != nullptr) {  // deterministic: per-CTA partials, summed in CTA order later
        float* pp = partials + static_cast<int64_t>(blockIdx.x) * 2 * d;
        *reinterpret_cast<float4*>(pp + c) = ds[j];
        *reinterpret_cast<float4*>(pp + d + c) = db[j];
      } else {
        atomicAdd(dscale + c, ds[j].x); atomicAdd(dscale + c + 1, ds[j].y);
        atomicAdd(dscale + c + 2, ds[j].z); atomicAdd(dscale + c + 3, ds[j].w);
        if (dbias != nullptr) {
          atomicAdd(dbias + c, db[j].x); atomicAdd(dbias + c + 1, db[j].y);
          atomicAdd(dbias + c + 2, db[j].z); atomicAdd(dbias + c + 3, db[j].w);
        }
      }
    }
  }
}



// Block-wide sum of four values with one shared-memory round (red >= 4 * warps floats).
__device__ __forceinline__ float4 block_sum4(float4 v, float* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v.x = warp_sum(v.x);
  v.y = warp_sum(v.y);
  v.z = warp_sum(v.z);
  v.w = warp_sum(v.w);
  __syncthreads();
  if (lane == 0) reinterpret_cast<float4*>(red)[w] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  float4 t = lane < nw ? reinterpret_cast<const float4*>(red)[lane] : make_float4(0.f, 0.f, 0.f, 0.f);
  t.x = warp_sum(t.x);
  t.y = warp_sum(t.y);
  t.z = warp_sum(t.z);
  t.w = warp_sum(t.w);
  return t;
}

// LayerNorm backward, two rows per step (d <= 1024 * V4, d % 4 == 0): both rows' x / dy loads
// are in flight together, their four row sums share one block reduction, and the residual
// gradient of both rows is prefetched into L1 before that reduction so its latency hides behind
// it. x / dy are kept in registers between the passes (no re-read).
// WG: also the column sums of the written residual gradient g_io (the bias gradient of the
// row-parallel projection whose output feeds this LayerNorm), as a third partial row.
template <int THREADS, int V4, typename DY, bool WG>
__global__ void __launch_bounds__(THREADS, 2) ln_bwd2_kernel(
    const float* __restrict__ x, const float* __restrict__ mean, const float* __restrict__ rstd,
    const float* __restrict__ scale, const DY* __restrict__ dy, float* __restrict__ g_io,
    bf16* __restrict__ g_bf16, float* __restrict__ dscale, float* __restrict__ dbias, int64_t M,
    int d, int accumulate, float* __restrict__ partials, int rms) {
  __shared__ __align__(16) float red[4 * (THREADS / 32)];
  float4 ds[V4], db[V4];
  // column sums of g_io live in shared memory ([j][thread] float4, conflict-free), not in
  // registers: the two-row kernel is at its register budget
  __shared__ float4 gsm[WG ? V4 * THREADS : 1];
  if constexpr (WG) {
#pragma unroll
    for (int j = 0; j < V4; ++j) gsm[j * THREADS + threadIdx.x] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int j = 0; j < V4; ++j) ds[j] = db[j] = make_float4(0, 0, 0, 0);
  const int64_t pairs = (M + 1) / 2;
  for (int64_t pr = blockIdx.x; pr < pairs; pr += gridDim.x) {
    const int64_t r0 = 2 * pr;
    const bool two = r0 + 1 < M;
    const int64_t r1 = two ? r0 + 1 : r0;
    const float mu0 = mean ? mean[r0] : 0.f, rs0 = rstd[r0], mu1 = mean ? mean[r1] : 0.f, rs1 = rstd[r1];
    float4 xa[V4], da[V4], xb[V4], dbv[V4];
#pragma unroll
    for (int j = 0; j < V4; ++j) {
      const int c = (threadIdx.x + j * THREADS) * 4;
      if (c < d) {
        xa[j] = __ldg(reinterpret_cast<const float4*>(x + r0 * d + c));
        da[j] = ldg4(dy + r0 * d + c);
        xb[j] = __ldg(reinterpret_cast<const float4*>(x + r1 * d + c));
        dbv[j] = ldg4(dy + r1 * d + c);
      }
    }
    if (accumulate && (threadIdx.x & 7) == 0) {  // one L1 prefetch per 128-byte line
#pragma unroll
      for (int j = 0; j < V4; ++j) {
        const int c = (threadIdx.x + j * THREADS) * 4;
        if (c < d) {
          asm volatile("prefetch.global.L1 [%0];" ::"l"(g_io + r0 * d + c));
          asm volatile("prefetch.global.L1 [%0];" ::"l"(g_io + r1 * d + c));
        }
      }
    }
    float4 sums = make_float4(0.f, 0.f, 0.f, 0.f);  // s1(row0), s2(row0), s1(row1), s2(row1)
#pragma unroll
    for (int j = 0; j < V4; ++j) {
      const int c = (threadIdx.x + j * THREADS) * 4;
      if (c < d) {
        const float4 sc = __ldg(reinterpret_cast<const float4*>(scale + c));
        const float4 ha = make_float4((xa[j].x - mu0) * rs0, (xa[j].y - mu0) * rs0, (xa[j].z - mu0) * rs0,
                                      (xa[j].w - mu0) * rs0);
        const float4 hb = make_float4((xb[j].x - mu1) * rs1, (xb[j].y - mu1) * rs1, (xb[j].z - mu1) * rs1,
                                      (xb[j].w - mu1) * rs1);
        ds[j].x += da[j].x * ha.x; ds[j].y += da[j].y * ha.y; ds[j].z += da[j].z * ha.z; ds[j].w += da[j].w * ha.w;
        db[j].x += da[j].x; db[j].y += da[j].y; db[j].z += da[j].z; db[j].w += da[j].w;
        if (two) {
          ds[j].x += dbv[j].x * hb.x; ds[j].y += dbv[j].y * hb.y; ds[j].z += dbv[j].z * hb.z; ds[j].w += dbv[j].w * hb.w;
          db[j].x += dbv[j].x; db[j].y += dbv[j].y; db[j].z += dbv[j].z; db[j].w += dbv[j].w;
        }
        const float gx = da[j].x * sc.x, gy = da[j].y * sc.y, gz = da[j].z * sc.z, gw = da[j].w * sc.w;
        sums.x += gx + gy + gz + gw;
        sums.y += gx * ha.x + gy * ha.y + gz * ha.z + gw * ha.w;
        const float hx = dbv[j].x * sc.x, hy = dbv[j].y * sc.y, hz = dbv[j].z * sc.z, hw = dbv[j].w * sc.w;
        sums.z += hx + hy + hz + hw;
        sums.w += hx * hb.x + hy * hb.y + hz * hb.z + hw * hb.w;
      }
    }
    const float4 t = block_sum4(sums, red);
    const float gm0 = rms ? 0.f : t.x / d, gxm0 = t.y / d, gm1 = rms ? 0.f : t.z / d, gxm1 = t.w / d;
#pragma unroll
    for (int j = 0; j < V4; ++j) {
      const int c = (threadIdx.x + j * THREADS) * 4;
      if (c < d) {
        const float4 sc = __ldg(reinterpret_cast<const float4*>(scale + c));
        float4 o;
        o.x = rs0 * (da[j].x * sc.x - gm0 - (xa[j].x - mu0) * rs0 * gxm0);
        o.y = rs0 * (da[j].y * sc.y - gm0 - (xa[j].y - mu0) * rs0 * gxm0);
        o.z = rs0 * (da[j].z * sc.z - gm0 - (xa[j].z - mu0) * rs0 * gxm0);
        o.w = rs0 * (da[j].w * sc.w - gm0 - (xa[j].w - mu0) * rs0 * gxm0);
        if (accumulate) {
          const float4 g = *reinterpret_cast<const float4*>(g_io + r0 * d + c);
          o.x += g.x; o.y += g.y; o.z += g.z; o.w += g.w;
        }
        *reinterpret_cast<float4*>(g_io + r0 * d + c) = o;
        float4 gacc;
        if constexpr (WG) gacc = o;
        uint2 w;
        w.x = dev::pack_bf16x2(o.x, o.y);
        w.y = dev::pack_bf16x2(o.z, o.w);
        *reinterpret_cast<uint2*>(g_bf16 + r0 * d + c) = w;
        if (two) {
          o.x = rs1 * (dbv[j].x * sc.x - gm1 - (xb[j].x - mu1) * rs1 * gxm1);
          o.y = rs1 * (dbv[j].y * sc.y - gm1 - (xb[j].y - mu1) * rs1 * gxm1);
          o.z = rs1 * (dbv[j].z * sc.z - gm1 - (xb[j].z - mu1) * rs1 * gxm1);
          o.w = rs1 * (dbv[j].w * sc.w - gm1 - (xb[j].w - mu1) * rs1 * gxm1);
          if (accumulate) {
            const float4 g = *reinterpret_cast<const float4*>(g_io + r1 * d + c);
            o.x += g.x; o.y += g.y; o.z += g.z; o.w += g.w;
          }
          *reinterpret_cast<float4*>(g_io + r1 * d + c) = o;
          if constexpr (WG) {
            gacc.x += o.x; gacc.y += o.y; gacc.z += o.z; gacc.w += o.w;
          }
          w.x = dev::pack_bf16x2(o.x, o.y);
          w.y = dev::pack_bf16x2(o.z, o.w);
          *reinterpret_cast<uint2*>(g_bf16 + r1 * d + c) = w;
        }
        if constexpr (WG) {
          float4 t = gsm[j * THREADS + threadIdx.x];
          t.x += gacc.x; t.y += gacc.y; t.z += gacc.z; t.w += gacc.w;
          gsm[j * THREADS + threadIdx.x] = t;
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < V4; ++j) {
    const int c = (threadIdx.x + j * THREADS) * 4;
    if (c < d) {
      if (partials != nullptr) {  // deterministic: per-CTA partials, summed in CTA order later
        float* pp = partials + static_cast<int64_t>(blockIdx.x) * (WG ? 3 : 2) * d;
        *reinterpret_cast<float4*>(pp + c) = ds[j];
        *reinterpret_cast<float4*>(pp + d + c) = db[j];
        if constexpr (WG) *reinterpret_cast<float4*>(pp + 2 * d + c) = gsm[j * THREADS + threadIdx.x];
      } else {
        atomicAdd(dscale + c, ds[j].x); atomicAdd(dscale + c + 1, ds[j].y);
        atomicAdd(dscale + c + 2, ds[j].z); atomicAdd(dscale + c + 3, ds[j].w);
        if (dbias != nullptr) {
          atomicAdd(dbias + c, db[j].x); atomicAdd(dbias + c + 1, db[j].y);
          atomicAdd(dbias + c + 2, db[j].z); atomicAdd(dbias + c + 3, db[j].w);
        }
      }
    }
  }
}



// dscale[c] += sum_b partials[b][0][c], dbias[c] += sum_b partials[b][1][c]: four interleaved
// accumulators (b mod 4) combined in a fixed order -- deterministic, and four loads in flight.
// Sum of the per-CTA LayerNorm parameter partials [nblk][2][d] in a fixed order (bit-identical
// on every replica): a CTA owns 32 columns; its 8 warps take interleaved row groups (coalesced
// 128-byte rows, 8x the loads in flight of one thread per column) and combine in warp order.
__global__ void __launch_bounds__(256) ln_param_reduce_kernel(const float* __restrict__ partials, int nblk, int d,
                                                              float* __restrict__ dscale, float* __restrict__ dbias,
                                                              int nsec, float* __restrict__ gsum) {
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;  // in [0, nsec * d)
  float s0 = 0.f, s1 = 0.f;
  if (c < nsec * d) {
    const int which = c / d, col = c - which * d;
    const float* src = partials + which * d + col;
    const int64_t stride = static_cast<int64_t>(nsec) * d;
    int b = w;
    for (; b + 8 < nblk; b += 16) {
      s0 += src[b * stride];
      s1 += src[(b + 8) * stride];
    }
    for (; b < nblk; b += 8) s0 += src[b * stride];
  }
  red[w][lane] = s0 + s1;
  __syncthreads();
  if (w == 0 && c < nsec * d) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red[i][lane];
    const int which = c / d, col = c - which * d;
    float* o = which == 0 ? dscale : which == 1 ? dbias : gsum;
    if (o != nullptr) o[col] += t;
  }
}

template <typename DY>
__global__ void ln_bwd_generic_kernel(const float* __restrict__ x, const float* __restrict__ mean,
                                      const float* __restrict__ rstd, const float* __restrict__ scale,
                                      const DY* __restrict__ dy, float* __restrict__ g_io,
                                      bf16* __restrict__ g_bf16, float* __restrict__ dscale,
                                      float* __restrict__ dbias, int d, int accumulate, int rms) {
  __shared__ float red[32];
  const int64_t row = blockIdx.x;
  const float mu = mean ? mean[row] : 0.f, rs = rstd[row];
  float s1 = 0.f, s2 = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float xh = (x[row * d + i] - mu) * rs;
    const float g = ld1(dy + row * d + i) * scale[i];
    s1 += g;
    s2 += g * xh;
  }
  const float gm = rms ? 0.f : block_sum(s1, red) / d;
  const float gxm = block_sum(s2, red) / d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float xh = (x[row * d + i] - mu) * rs;
    const float dv = ld1(dy + row * d + i);
    const float g = dv * scale[i];
    float dx = rs * (g - gm - xh * gxm);
    if (accumulate) dx += g_io[row * d + i];
    g_io[row * d + i] = dx;
    g_bf16[row * d + i] = __float2bfloat16(dx);
    atomicAdd(dscale + i, dv * xh);
    if (dbias != nullptr) atomicAdd(dbias + i, dv);
  }
}

// ------------------------------------------------------------------------------------------
// column sums (bias gradients)
// ------------------------------------------------------------------------------------------
constexpr int kColChunk = 64;  // columns per CTA
constexpr int kRowChunk = 256; // rows per CTA (partials)

template <typename T>
__device__ __forceinline__ float ld_as_float(const T* p);
template <>
__device__ __forceinline__ float ld_as_float<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ld_as_float<bf16>(const bf16* p) { return __bfloat162float(*p); }

// stage 1: partial[chunk][n] = sum over the chunk's 256 rows. A CTA covers 256 columns:
// 32 column groups of 8 (one 16-byte bf16 load / two float4 loads each) x 8 row lanes.
template <typename T>
__device__ __forceinline__ void load8(const T* p, float (&v)[8]);
template <>
__device__ __forceinline__ void load8<bf16>(const bf16* p, float (&v)[8]) {
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = dev::unpack_bf16x2(w[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
template <>
__device__ __forceinline__ void load8<float>(const float* p, float (&v)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p + 4));
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

template <typename T>
__global__ void __launch_bounds__(256) colsum_partial_kernel(const T* __restrict__ X, int64_t ld, int64_t M, int N,
                                                             float* __restrict__ partial) {
  __shared__ float sm[8][257];
  const int cg = threadIdx.x & 31;  // column group
  const int rl = threadIdx.x >> 5;  // row lane
  const int c0 = blockIdx.x * 256 + cg * 8;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kRowChunk;
  const int64_t r_end = (M < r0 + kRowChunk) ? M : r0 + kRowChunk;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (c0 + 8 <= N) {
    for (int64_t r = r0 + rl; r < r_end; r += 8) {
      float v[8];
      load8<T>(X + r * ld + c0, v);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += v[i];
    }
  } else {
    for (int64_t r = r0 + rl; r < r_end; r += 8)
      for (int i = 0; i < 8 && c0 + i < N; ++i) acc[i] += ld_as_float(X + r * ld + c0 + i);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) sm[rl][cg * 8 + i] = acc[i];
  __syncthreads();
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c < N) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sm[k][threadIdx.x];
    partial[static_cast<int64_t>(blockIdx.y) * N + c] = t;
  }
}

// out[n] (+)= sum over chunks of partial[c][n] in a fixed order (per-32-row partials written by
// the GeLU-backward GEMM epilogue): 32 columns x 8 chunk lanes per CTA, then a fixed-order fold.
__global__ void __launch_bounds__(256) colsum_chunks_kernel(const float* __restrict__ partial, int chunks, int N,
                                                            int seg, float* out0, float* out1, float* out2,
                                                            int accumulate) {
  __shared__ float sm[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int n = blockIdx.x * 32 + tx;
  float s = 0.f;
  if (n < N) {
    for (int c = ty; c < chunks; c += 8) s += partial[static_cast<int64_t>(c) * N + n];
  }
  sm[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && n < N) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += sm[i][tx];
    const int si = n / seg;
    float* o = (si == 0 ? out0 : si == 1 ? out1 : out2) + (n - si * seg);
    *o = accumulate ? *o + t : t;
  }
}

__global__ void colsum_final_kernel(const float* __restrict__ partial, int chunks, int N, int seg,
                                    float* out0, float* out1, float* out2, int accumulate) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  float s = 0.f;
  for (int c = 0; c < chunks; ++c) s += partial[static_cast<int64_t>(c) * N + n];
  const int si = n / seg;
  float* o = (si == 0 ? out0 : si == 1 ? out1 : out2) + (n - si * seg);
  *o = accumulate ? *o + s : s;
}

// ------------------------------------------------------------------------------------------
// reductions / cross entropy
// ------------------------------------------------------------------------------------------
__global__ void sum_f32_kernel(const float* __restrict__ x, int64_t n, float* out) {
  __shared__ float red[32];
  float s = 0.f;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

__global__ void loss_reduce_kernel(const float* __restrict__ wl, int64_t n, const float* wsum,
                                   double* loss, int* gate) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += wl[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (blockDim.x + 31) / 32; ++w) t += red[w];
    const double l = t / static_cast<double>(*wsum);
    *loss = l;
    if (gate != nullptr && !isfinite(l)) atomicOr(gate, 2);
  }
}

// One CTA per row. Pass 1: per-thread online (max, sumexp) -> block combine. Pass 2: gradient.
__global__ void __launch_bounds__(512) xent_kernel(bf16* __restrict__ logits, int64_t ld, int V,
                                                   const int32_t* __restrict__ targets,
                                                   const float* __restrict__ weights,
                                                   const float* __restrict__ wsum,
                                                   float* __restrict__ wloss, int write_grad) {
  __shared__ float red_m[32], red_s[32];
  __shared__ float bc[2];
  const int64_t row = blockIdx.x;
  bf16* lr = logits + row * ld;
  const bool vec = (V % 8 == 0) && (ld % 8 == 0);
  float mx = -INFINITY, se = 0.f;
  auto acc = [&](float x) {
    if (x > mx) {
      se = se * __expf(mx - x) + 1.f;
      mx = x;
    } else {
      se += __expf(x - mx);
    }
  };
  if (vec) {
    for (int i = threadIdx.x * 8; i < V; i += blockDim.x * 8) {
      const uint4 u = *reinterpret_cast<const uint4*>(lr + i);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = dev::unpack_bf16x2(w[j]);
        acc(f.x);
        acc(f.y);
      }
    }
  } else {
    for (int i = threadIdx.x; i < V; i += blockDim.x) acc(__bfloat162float(lr[i]));
  }
  // combine (max, sum) across the warp then the block
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, mx, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, se, o);
    const float m = fmaxf(mx, m2);
    se = (mx == -INFINITY ? 0.f : se * __expf(mx - m)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - m));
    mx = m;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    red_m[wid] = mx;
    red_s[wid] = se;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = -INFINITY;
    const int nw = blockDim.x / 32;
    for (int w = 0; w < nw; ++w) m = fmaxf(m, red_m[w]);
    float s = 0.f;
    for (int w = 0; w < nw; ++w) s += red_s[w] * __expf(red_m[w] - m);
    bc[0] = m;
    bc[1] = s;
    const int tgt = targets[row];
    const float lse = m + logf(s);
    wloss[row] = weights[row] * (lse - __bfloat162float(lr[tgt]));
  }
  __syncthreads();
  if (!write_grad) return;
  const float m = bc[0];
  const float inv = 1.0f / bc[1];
  const float scale = weights[row] / *wsum;
  const int tgt = targets[row];
  if (vec) {
    for (int i = threadIdx.x * 8; i < V; i += blockDim.x * 8) {
      uint4 u = *reinterpret_cast<const uint4*>(lr + i);
      uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = dev::unpack_bf16x2(w[j]);
        float a = __expf(f.x - m) * inv, b = __expf(f.y - m) * inv;
        if (i + 2 * j == tgt) a -= 1.f;
        if (i + 2 * j + 1 == tgt) b -= 1.f;
        w[j] = dev::pack_bf16x2(a * scale, b * scale);
      }
      *reinterpret_cast<uint4*>(lr + i) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  } else {
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
      float a = __expf(__bfloat162float(lr[i]) - m) * inv;
      if (i == tgt) a -= 1.f;
      lr[i] = __float2bfloat16(a * scale);
    }
  }
}

// ---- vocab-parallel cross entropy ----
__global__ void __launch_bounds__(512) xent_vp_stats_kernel(const bf16* __restrict__ logits, int64_t ld, int Vl,
                                                            int v0, const int32_t* __restrict__ targets,
                                                            float* __restrict__ stats, float* __restrict__ tlogit) {
  __shared__ float red_m[32], red_s[32];
  const int64_t row = blockIdx.x;
  const bf16* lr = logits + row * ld;
  float mx = -INFINITY, se = 0.f;
  for (int i = threadIdx.x; i < Vl; i += blockDim.x) {
    const float x = __bfloat162float(lr[i]);
    if (x > mx) {
      se = se * __expf(mx - x) + 1.f;
      mx = x;
    } else {
      se += __expf(x - mx);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, mx, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, se, o);
    const float m = fmaxf(mx, m2);
    se = (mx == -INFINITY ? 0.f : se * __expf(mx - m)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - m));
    mx = m;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    red_m[wid] = mx;
    red_s[wid] = se;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = -INFINITY;
    const int nw = blockDim.x / 32;
    for (int w = 0; w < nw; ++w) m = fmaxf(m, red_m[w]);
    float sum = 0.f;
    for (int w = 0; w < nw; ++w) sum += red_s[w] * __expf(red_m[w] - m);
    stats[2 * row] = m;
    stats[2 * row + 1] = sum;
    const int t = targets[row] - v0;
    tlogit[row] = (t >= 0 && t < Vl) ? __bfloat162float(lr[t]) : 0.f;
  }
}

__global__ void xent_vp_combine_kernel(const float* __restrict__ stats_all, int t, int64_t M,
                                       const float* __restrict__ tlogit, const float* __restrict__ weights,
                                       float* __restrict__ lse, float* __restrict__ wloss) {
  for (int64_t m = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; m < M;
       m += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float mx = -INFINITY;
    for (int r = 0; r < t; ++r) mx = fmaxf(mx, stats_all[(r * M + m) * 2]);
    float s = 0.f;
    for (int r = 0; r < t; ++r) s += stats_all[(r * M + m) * 2 + 1] * __expf(stats_all[(r * M + m) * 2] - mx);
    const float l = mx + logf(s);
    lse[m] = l;
    wloss[m] = weights[m] * (l - tlogit[m]);
  }
}

__global__ void __launch_bounds__(512) xent_vp_grad_kernel(bf16* __restrict__ logits, int64_t ld, int Vl, int v0,
                                                           const int32_t* __restrict__ targets,
                                                           const float* __restrict__ lse,
                                                           const float* __restrict__ weights,
                                                           const float* __restrict__ wsum) {
  const int64_t row = blockIdx.x;
  bf16* lr = logits + row * ld;
  const float l = lse[row];
  const float scale = weights[row] / *wsum;
  const int t = targets[row] - v0;
  for (int i = threadIdx.x; i < Vl; i += blockDim.x) {
    float a = __expf(__bfloat162float(lr[i]) - l);
    if (i == t) a -= 1.f;
    lr[i] = __float2bfloat16(a * scale);
  }
}

__global__ void add_residual_bias_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                         const float* __restrict__ bias, float* __restrict__ y,
                                         int64_t n4, int d) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 x = reinterpret_cast<const float4*>(a)[i];
    const float4 z = reinterpret_cast<const float4*>(b)[i];
    const int c = static_cast<int>((i * 4) % d);
    const float4 bb = bias ? *reinterpret_cast<const float4*>(bias + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    reinterpret_cast<float4*>(y)[i] = make_float4(x.x + z.x + bb.x, x.y + z.y + bb.y, x.z + z.z + bb.z, x.w + z.w + bb.w);
  }
}

__global__ void add_residual_bias_bf16_kernel(const float* __restrict__ a, const bf16* __restrict__ b,
                                              const float* __restrict__ bias, float* __restrict__ y, int64_t n4,
                                              int d) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 x = reinterpret_cast<const float4*>(a)[i];
    const float4 z = ldg4(b + i * 4);
    const int c = static_cast<int>((i * 4) % d);
    const float4 bb = bias ? *reinterpret_cast<const float4*>(bias + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    reinterpret_cast<float4*>(y)[i] = make_float4(x.x + z.x + bb.x, x.y + z.y + bb.y, x.z + z.z + bb.z, x.w + z.w + bb.w);
  }
}

// ------------------------------------------------------------------------------------------
// optimizer / misc
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void adamw_one(float& p, float& m, float& v, float g, float lr, float b1,
                                          float b2, float eps, float wd, float c1, float c2) {
  dev::adamw_update(p, m, v, g, lr, b1, b2, eps, wd, c1, c2);
}

__global__ void adamw_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                             const float* __restrict__ g, bf16* __restrict__ shadow, int64_t n,
                             float lr, float b1, float b2, float eps, float wd, float c1, float c2,
                             const int* __restrict__ gate) {
  if (gate != nullptr && *gate != 0) return;  // a non-finite loss or gradient: state unchanged
  const int64_t n4 = n / 4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4; i += stride) {
    float4 pp = reinterpret_cast<float4*>(p)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    const float4 gg = reinterpret_cast<const float4*>(g)[i];
    adamw_one(pp.x, mm.x, vv.x, gg.x, lr, b1, b2, eps, wd, c1, c2);
    adamw_one(pp.y, mm.y, vv.y, gg.y, lr, b1, b2, eps, wd, c1, c2);
    adamw_one(pp.z, mm.z, vv.z, gg.z, lr, b1, b2, eps, wd, c1, c2);
    adamw_one(pp.w, mm.w, vv.w, gg.w, lr, b1, b2, eps, wd, c1, c2);
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    uint2 w;
    w.x = dev::pack_bf16x2(pp.x, pp.y);
    w.y = dev::pack_bf16x2(pp.z, pp.w);
    reinterpret_cast<uint2*>(shadow)[i] = w;
  }
  for (int64_t i = n4 * 4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    adamw_one(p[i], m[i], v[i], g[i], lr, b1, b2, eps, wd, c1, c2);
    shadow[i] = __float2bfloat16(p[i]);
  }
}

__global__ void nonfinite_kernel(const float* __restrict__ x, int64_t n, int* flag) {
  int bad = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    bad |= !isfinite(x[i]);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

__global__ void scale_kernel(float* x, int64_t n, float a) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    x[i] *= a;
  }
}

__global__ void cast_kernel(const float* __restrict__ x, bf16* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    y[i] = __float2bfloat16(x[i]);
  }
}

__global__ void widen_kernel(const bf16* __restrict__ x, float* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    y[i] = __bfloat162float(x[i]);
  }
}

__global__ void fill_kernel(float* x, int64_t n, float v) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    x[i] = v;
  }
}

struct RankPtrs {
  float* p[16];
};

__global__ void sum_ranks_kernel(RankPtrs bufs, int nranks, int64_t n, float scale) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float s = bufs.p[0][i];
    for (int r = 1; r < nranks; ++r) s += bufs.p[r][i];
    s *= scale;
    for (int r = 0; r < nranks; ++r) bufs.p[r][i] = s;
  }
}

struct RankPtrsBf16 {
  bf16* p[16];
};

// bf16 payloads: fp32 sum in ascending rank order, one rounding (NCCL's ring rounds per hop)
__global__ void sum_ranks_bf16_kernel(RankPtrsBf16 bufs, int nranks, int64_t n, float scale) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float s = __bfloat162float(bufs.p[0][i]);
    for (int r = 1; r < nranks; ++r) s += __bfloat162float(bufs.p[r][i]);
    const bf16 o = __float2bfloat16(s * scale);
    for (int r = 0; r < nranks; ++r) bufs.p[r][i] = o;
  }
}

__device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void init_normal_kernel(float* out, int64_t lr, int64_t lc, int64_t r0, int64_t c0,
                                   int64_t cols, uint64_t key, uint64_t base, double scale) {
  const int64_t n = lr * lc;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / lc, j = e - (e / lc) * lc;
    const uint64_t g = static_cast<uint64_t>((r0 + i) * cols + (c0 + j));
    const uint64_t d1 = splitmix_mix(key + base + 2 * g);
    const uint64_t d2 = splitmix_mix(key + base + 2 * g + 1);
    double u1 = static_cast<double>(d1 >> 11) * 0x1.0p-53;
    const double u2 = static_cast<double>(d2 >> 11) * 0x1.0p-53;
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    const double z = r * cos(2.0 * 3.14159265358979323846 * u2);
    out[e] = static_cast<float>(z * scale);
  }
}

}  // namespace

// ------------------------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------------------------
void embed_fwd(const int32_t* ids, const float* tok, const float* pos, float* h, int64_t M, int T,
               int d, cudaStream_t s) {
  embed_fwd_kernel<<<static_cast<unsigned>(M), d >= 1024 ? 256 : 128, 0, s>>>(ids, tok, pos, h, T, d);
}

void embed_bwd_tok(const int32_t* ids, const float* g, float* dtok, int64_t M, int d, int V, uint32_t* keys,
                   cudaStream_t s) {
  if (keys == nullptr || M > 32768 || V > 65535 || d % 4 != 0) {
    embed_bwd_tok_kernel<<<static_cast<unsigned>(M), 256, 0, s>>>(ids, g, dtok, d);
    return;
  }
  const int n = static_cast<int>(embed_bwd_keys(M));
  static int configured_bytes = 0;
  if (n * 4 > configured_bytes) {
    cudaFuncSetAttribute(sort_token_keys_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, n * 4);
    configured_bytes = n * 4;
  }
  sort_token_keys_kernel<<<1, 1024, n * 4, s>>>(ids, M, n, keys);
  const int64_t per = 16;
  embed_accum_sorted_kernel<<<static_cast<unsigned>((M + per - 1) / per), 256, 0, s>>>(keys, M, g, dtok, d, per);
}

int64_t embed_bwd_keys(int64_t M) {
  int64_t n = 1;
  while (n < M) n <<= 1;
  return n < 2 ? 2 : n;
}

void embed_bwd_pos(const float* g, float* dpos, int B, int T, int d, int accumulate, cudaStream_t s) {
  embed_bwd_pos_kernel<<<T, 256, 0, s>>>(g, dpos, B, T, d, accumulate);
}

// Decode-size rows (M <= 8, one CTA of 1024 threads per row): the statistics in one pass (sum and
// sum of squares reduced together, var = E[x^2] - mean^2), so the row costs one block reduction
// instead of two -- the kernel is latency-bound at this size. SW_DECODE_LN1P=0 keeps ln_fwd.
template <int V4>
__global__ void __launch_bounds__(1024) ln_fwd_1pass_kernel(const float* __restrict__ x, const float* __restrict__ scale,
                                                            const float* __restrict__ bias, bf16* __restrict__ y,
                                                            float* __restrict__ mean_out, float* __restrict__ rstd_out,
                                                            int d, float eps, int rms) {
  asm volatile("griddepcontrol.launch_dependents;");  // the next weight-streaming GEMM may start
  // launched as a programmatic dependent (decode): x comes from the kernel before
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ float2 red[32];
  const int64_t row = blockIdx.x;
  const float* xr = x + row * d;
  float4 v[V4];
  float s = 0.f, q = 0.f;
#pragma unroll
  for (int j = 0; j < V4; ++j) {
    const int c = (threadIdx.x + j * 1024) * 4;
    v[j] = c < d ? *reinterpret_cast<const float4*>(xr + c) : make_float4(0, 0, 0, 0);
    s += v[j].x + v[j].y + v[j].z + v[j].w;
    q += v[j].x * v[j].x + v[j].y * v[j].y + v[j].z * v[j].z + v[j].w * v[j].w;
  }
  s = warp_sum(s);
  q = warp_sum(q);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = make_float2(s, q);
  __syncthreads();
  float2 t = red[lane];
  t.x = warp_sum(t.x);
  t.y = warp_sum(t.y);
  const float mean = rms ? 0.f : t.x / d;
  const float var = fmaxf(t.y / d - mean * mean, 0.f);
  const float rstd = 1.0f / sqrtf(var + eps);
  bf16* yr = y + row * d;
#pragma unroll
  for (int j = 0; j < V4; ++j) {
    const int c = (threadIdx.x + j * 1024) * 4;
    if (c < d) {
      const float4 sc = *reinterpret_cast<const float4*>(scale + c);
      const float4 bi = rms ? make_float4(0.f, 0.f, 0.f, 0.f) : *reinterpret_cast<const float4*>(bias + c);
      uint2 o;
      o.x = dev::pack_bf16x2((v[j].x - mean) * rstd * sc.x + bi.x, (v[j].y - mean) * rstd * sc.y + bi.y);
      o.y = dev::pack_bf16x2((v[j].z - mean) * rstd * sc.z + bi.z, (v[j].w - mean) * rstd * sc.w + bi.w);
      *reinterpret_cast<uint2*>(yr + c) = o;
    }
  }
  if (threadIdx.x == 0) {
    if (mean_out != nullptr) mean_out[row] = mean;
    rstd_out[row] = rstd;
  }
}

void layernorm_fwd_small(const float* x, const float* scale, const float* bias, bf16* y, float* mean, float* rstd,
                         int64_t M, int d, float eps, cudaStream_t s, int rms) {
  static const bool on = [] {
    const char* e = std::getenv("SW_DECODE_LN1P");
    return !(e != nullptr && e[0] == '0');
  }();
  const unsigned g = static_cast<unsigned>(M);
  static const bool pdl = [] {
    const char* e = std::getenv("SW_DECODE_PDL");
    return !(e != nullptr && e[0] == '0');
  }();
  if (on && M <= 8 && d % 4 == 0 && d <= 12288) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g);
    cfg.blockDim = dim3(1024);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (d <= 4096) {
      cudaLaunchKernelEx(&cfg, ln_fwd_1pass_kernel<1>, x, scale, bias, y, mean, rstd, d, eps, rms);
    } else {
      cudaLaunchKernelEx(&cfg, ln_fwd_1pass_kernel<3>, x, scale, bias, y, mean, rstd, d, eps, rms);
    }
  } else {
    layernorm_fwd(x, scale, bias, y, mean, rstd, M, d, eps, s, rms);
  }
}

void layernorm_fwd(const float* x, const float* scale, const float* bias, bf16* y, float* mean,
                   float* rstd, int64_t M, int d, float eps, cudaStream_t s, int rms) {
  const unsigned g = static_cast<unsigned>(M);
  if (d % 4 == 0 && d <= 512) {
    ln_fwd_kernel<32, 4><<<g, 32, 0, s>>>(x, scale, bias, y, mean, rstd, d, eps, rms);
  } else if (d % 4 == 0 && d <= 4096) {
    ln_fwd_kernel<256, 4><<<g, 256, 0, s>>>(x, scale, bias, y, mean, rstd, d, eps, rms);
  } else if (d % 4 == 0 && d <= 12288) {
    ln_fwd_kernel<512, 6><<<g, 512, 0, s>>>(x, scale, bias, y, mean, rstd, d, eps, rms);
  } else {
    ln_fwd_generic_kernel<<<g, 256, 0, s>>>(x, scale, bias, y, mean, rstd, d, eps, rms);
  }
}

// SW_LN_BWD_V1=1 selects the one-row-per-step kernel (A/B comparisons).
static bool ln_bwd_v1() {
  static const bool v1 = [] {
    const char* e = std::getenv("SW_LN_BWD_V1");
    return e != nullptr && e[0] == '1';
  }();
  return v1;
}

int64_t layernorm_bwd_partials(int d) { return static_cast<int64_t>(4 * kSMs) * 2 * d; }

template <typename DY>
static void layernorm_bwd_t(const float* x, const float* mean, const float* rstd, const float* scale, const DY* dy,
                            float* g_io, bf16* g_bf16, float* dscale, float* dbias, int64_t M, int d, int accumulate,
                            cudaStream_t s, float* partials, int rms, float* gsum) {
  bool gsum_fused = false;
  const unsigned g = static_cast<unsigned>(M < 4 * kSMs ? M : 4 * kSMs);
  unsigned nblk = g;
  if (d % 4 == 0 && d <= 512) {
    ln_bwd_kernel<32, 4, DY><<<g, 32, 0, s>>>(x, mean, rstd, scale, dy, g_io, g_bf16, dscale, dbias, M, d, accumulate,
                                          partials, rms);
  } else if (d % 4 == 0 && d <= 4096 && ln_bwd_v1()) {
    ln_bwd_kernel<256, 4, DY><<<g, 256, 0, s>>>(x, mean, rstd, scale, dy, g_io, g_bf16, dscale, dbias, M, d, accumulate,
                                            partials, rms);
  } else if (d % 4 == 0 && d <= 4096) {
    const unsigned g2 = static_cast<unsigned>((M + 1) / 2 < 2 * kSMs ? (M + 1) / 2 : 2 * kSMs);
    nblk = g2;
    if (gsum != nullptr && partials != nullptr) {
      gsum_fused = true;
      ln_bwd2_kernel<256, 4, DY, true><<<g2, 256, 0, s>>>(x, mean, rstd, scale, dy, g_io, g_bf16, dscale, dbias, M, d,
                                                          accumulate, partials, rms);
    } else {
      ln_bwd2_kernel<256, 4, DY, false><<<g2, 256, 0, s>>>(x, mean, rstd, scale, dy, g_io, g_bf16, dscale, dbias, M, d,
                                                           accumulate, partials, rms);
    }
  } else if (d % 4 == 0 && d <= 12288) {
    ln_bwd_kernel<512, 6, DY><<<g, 512, 0, s>>>(x, mean, rstd, scale, dy, g_io, g_bf16, dscale, dbias, M, d, accumulate,
                                            partials, rms);
  } else {
    // one CTA per row: parameter partials would be row-sized; this shape keeps the atomics
    ln_bwd_generic_kernel<DY><<<static_cast<unsigned>(M), 256, 0, s>>>(x, mean, rstd, scale, dy, g_io, g_bf16,
                                                                  dscale, dbias, d, accumulate, rms);
    return;
  }
  if (partials != nullptr) {
    const int nsec = gsum_fused ? 3 : 2;
    ln_param_reduce_kernel<<<static_cast<unsigned>((nsec * d + 31) / 32), 256, 0, s>>>(
        partials, static_cast<int>(nblk), d, dscale, dbias, nsec, gsum_fused ? gsum : nullptr);
  }
  if (gsum != nullptr && !gsum_fused) {
    if (partials == nullptr) throw std::runtime_error("layernorm_bwd: column sums need the partials scratch");
    colsum_f32(g_io, d, M, d, gsum, 1, partials, s);
  }
}

void layernorm_bwd(const float* x, const float* mean, const float* rstd, const float* scale, const float* dy,
                   float* g_io, bf16* g_bf16, float* dscale, float* dbias, int64_t M, int d, int accumulate,
                   cudaStream_t s, float* partials, int rms, float* gsum) {
  layernorm_bwd_t(x, mean, rstd, scale, dy, g_io, g_bf16, dscale, dbias, M, d, accumulate, s, partials, rms, gsum);
}

void layernorm_bwd(const float* x, const float* mean, const float* rstd, const float* scale, const bf16* dy,
                   float* g_io, bf16* g_bf16, float* dscale, float* dbias, int64_t M, int d, int accumulate,
                   cudaStream_t s, float* partials, int rms, float* gsum) {
  layernorm_bwd_t(x, mean, rstd, scale, dy, g_io, g_bf16, dscale, dbias, M, d, accumulate, s, partials, rms, gsum);
}

void colsum_bf16(const bf16* X, int64_t ld, int64_t M, int N, int seg, float* out0, float* out1,
                 float* out2, int accumulate, float* scratch, cudaStream_t s) {
  const int chunks = static_cast<int>((M + kRowChunk - 1) / kRowChunk);
  dim3 grid((N + 255) / 256, chunks);
  colsum_partial_kernel<bf16><<<grid, 256, 0, s>>>(X, ld, M, N, scratch);
  colsum_final_kernel<<<(N + 255) / 256, 256, 0, s>>>(scratch, chunks, N, seg > 0 ? seg : N, out0,
                                                     out1, out2, accumulate);
}

void colsum_chunks(const float* partial, int chunks, int N, float* out, int accumulate, cudaStream_t s, int seg,
                   float* out1, float* out2) {
  colsum_chunks_kernel<<<(N + 31) / 32, 256, 0, s>>>(partial, chunks, N, seg > 0 ? seg : N, out, out1, out2,
                                                     accumulate);
}

void colsum_f32(const float* X, int64_t ld, int64_t M, int N, float* out, int accumulate,
                float* scratch, cudaStream_t s) {
  const int chunks = static_cast<int>((M + kRowChunk - 1) / kRowChunk);
  dim3 grid((N + 255) / 256, chunks);
  colsum_partial_kernel<float><<<grid, 256, 0, s>>>(X, ld, M, N, scratch);
  colsum_final_kernel<<<(N + 255) / 256, 256, 0, s>>>(scratch, chunks, N, N, out, nullptr, nullptr,
                                                     accumulate);
}

void sum_f32(const float* x, int64_t n, float* out, cudaStream_t s) {
  sum_f32_kernel<<<1, 1024, 0, s>>>(x, n, out);
}

void xent_fwd_bwd(bf16* logits, int64_t ld, int64_t M, int V, const int32_t* targets,
                  const float* weights, const float* wsum, float* wloss, int write_grad,
                  cudaStream_t s) {
  xent_kernel<<<static_cast<unsigned>(M), 512, 0, s>>>(logits, ld, V, targets, weights, wsum, wloss,
                                                       write_grad);
}

void xent_vp_stats(const bf16* logits, int64_t ld, int64_t M, int Vl, int v0, const int32_t* targets,
                   float* stats, float* tlogit, cudaStream_t s) {
  xent_vp_stats_kernel<<<static_cast<unsigned>(M), 512, 0, s>>>(logits, ld, Vl, v0, targets, stats, tlogit);
}

void xent_vp_combine(const float* stats_all, int t, int64_t M, const float* tlogit, const float* weights,
                     float* lse, float* wloss, cudaStream_t s) {
  xent_vp_combine_kernel<<<grid_for(M, 256), 256, 0, s>>>(stats_all, t, M, tlogit, weights, lse, wloss);
}

void xent_vp_grad(bf16* logits, int64_t ld, int64_t M, int Vl, int v0, const int32_t* targets, const float* lse,
                  const float* weights, const float* wsum, cudaStream_t s) {
  xent_vp_grad_kernel<<<static_cast<unsigned>(M), 512, 0, s>>>(logits, ld, Vl, v0, targets, lse, weights, wsum);
}

void loss_reduce(const float* wloss, int64_t M, const float* wsum, double* loss, cudaStream_t s, int* gate) {
  loss_reduce_kernel<<<1, 1024, 0, s>>>(wloss, M, wsum, loss, gate);
}

void add_residual_bias(const float* a, const float* b, const float* bias, float* y, int64_t M,
                       int d, cudaStream_t s) {
  const int64_t n4 = M * d / 4;
  add_residual_bias_kernel<<<grid_for(n4, 256), 256, 0, s>>>(a, b, bias, y, n4, d);
}

void add_residual_bias(const float* a, const bf16* b, const float* bias, float* y, int64_t M, int d,
                       cudaStream_t s) {
  const int64_t n4 = M * d / 4;
  add_residual_bias_bf16_kernel<<<grid_for(n4, 256), 256, 0, s>>>(a, b, bias, y, n4, d);
}

void adamw(float* p, float* m, float* v, const float* g, bf16* shadow, int64_t n, float lr,
           float b1, float b2, float eps, float wd, float c1, float c2, cudaStream_t s, const int* gate) {
  adamw_kernel<<<grid_for(n / 4 + 1, 256), 256, 0, s>>>(p, m, v, g, shadow, n, lr, b1, b2, eps, wd, c1, c2, gate);
}

void nonfinite_check(const float* x, int64_t n, int* flag, cudaStream_t s) {
  nonfinite_kernel<<<grid_for(n, 256, 4), 256, 0, s>>>(x, n, flag);
}

void scale_f32(float* x, int64_t n, float a, cudaStream_t s) {
  scale_kernel<<<grid_for(n, 256, 4), 256, 0, s>>>(x, n, a);
}

void cast_f32_bf16(const float* x, bf16* y, int64_t n, cudaStream_t s) {
  cast_kernel<<<grid_for(n, 256, 4), 256, 0, s>>>(x, y, n);
}

void cast_bf16_f32(const bf16* x, float* y, int64_t n, cudaStream_t s) {
  widen_kernel<<<grid_for(n, 256, 4), 256, 0, s>>>(x, y, n);
}

void fill_f32(float* out, int64_t n, float v, cudaStream_t s) {
  fill_kernel<<<grid_for(n, 256, 4), 256, 0, s>>>(out, n, v);
}

void sum_ranks_f32(float* const* bufs, int nranks, int64_t n, float scale, cudaStream_t s) {
  RankPtrs p{};
  for (int r = 0; r < nranks && r < 16; ++r) p.p[r] = bufs[r];
  sum_ranks_kernel<<<grid_for(n, 256, 4), 256, 0, s>>>(p, nranks, n, scale);
}

void sum_ranks_bf16(bf16* const* bufs, int nranks, int64_t n, float scale, cudaStream_t s) {
  RankPtrsBf16 p{};
  for (int r = 0; r < nranks && r < 16; ++r) p.p[r] = bufs[r];
  sum_ranks_bf16_kernel<<<grid_for(n, 256, 4), 256, 0, s>>>(p, nranks, n, scale);
}

void init_normal(float* out, int64_t lr, int64_t lc, int64_t r0, int64_t c0, int64_t cols,
                 uint64_t key, uint64_t base_counter, double scale, cudaStream_t s) {
  init_normal_kernel<<<grid_for(lr * lc, 256, 4), 256, 0, s>>>(out, lr, lc, r0, c0, cols, key,
                                                              base_counter, scale);
}

}  // namespace k
}  // namespace sw
