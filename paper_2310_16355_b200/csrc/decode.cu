// Greedy-decode kernels (the Predictor's next-token loop, cli.cpp:425-447,
// with a KV cache instead of re-running the window): one new position per sequence per step.
// HBM-bound (every step reads the weights and the cached keys/values once).
#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "kernels.h"
#include "sm100.cuh"

namespace sw {
namespace k {

namespace {

// x[b] = tok[ids[b]] + pos[p]   (model.hpp:92 embedding + learned position)
__global__ void embed_rows_kernel(const int32_t* __restrict__ ids, const float* __restrict__ tok,
                                  const float* __restrict__ pos, int p, const int* __restrict__ pd,
                                  float* __restrict__ x, int d) {
  if (pd != nullptr) p = *pd;  // position kept on the device (CUDA-graph decode steps)
  const int b = blockIdx.x;
  const int64_t id = ids[b];
  for (int c = threadIdx.x; c < d; c += blockDim.x) x[static_cast<int64_t>(b) * d + c] = tok[id * d + c] + pos[static_cast<int64_t>(p) * d + c];
}

// k | v of the new row b go to cache row b*T + p of the layer's qkv activations
__global__ void kv_scatter_kernel(const bf16* __restrict__ src, bf16* __restrict__ cache, int T, int p,
                                  const int* __restrict__ pd, int dl) {
  if (pd != nullptr) p = *pd;
  const int b = blockIdx.x;
  const bf16* s = src + static_cast<int64_t>(b) * 3 * dl + dl;
  bf16* t = cache + (static_cast<int64_t>(b) * T + p) * 3 * dl + dl;
  for (int c = threadIdx.x * 8; c < 2 * dl; c += blockDim.x * 8) {
    *reinterpret_cast<uint4*>(t + c) = *reinterpret_cast<const uint4*>(s + c);
  }
}

// One CTA per (sequence, head): the new query against cached keys 0..p (causal). Lanes work in
// groups of G = hd/8 (8 head-dim elements each, 16-byte loads of k and v); a warp handles 32/G
// keys per step with an online softmax per group; groups and warps merge through shared memory.
template <int HD>
__global__ void __launch_bounds__(256) decode_attention_kernel(const bf16* __restrict__ qnew,
                                                               const bf16* __restrict__ cache,
                                                               bf16* __restrict__ out, int T, int p,
                                                               const int* __restrict__ pd, int Hl,
                                                               float scale_log2) {
  if (pd != nullptr) p = *pd;
  constexpr int G = HD / 8;          // lanes per key
  constexpr int KPW = 32 / G;        // keys per warp step
  constexpr int NG = 8 * KPW;        // groups per CTA
  __shared__ float sm_m[NG], sm_l[NG];
  __shared__ float sm_o[NG][HD];
  const int b = blockIdx.x / Hl, h = blockIdx.x % Hl;
  const int dl = Hl * HD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / G, gl = lane % G;
  const int gid = warp * KPW + grp;
  float q[8];
  {
    const uint4 qv = *reinterpret_cast<const uint4*>(qnew + static_cast<int64_t>(b) * 3 * dl + h * HD + gl * 8);
    const uint32_t qq[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = dev::unpack_bf16x2(qq[e]);
      q[2 * e] = f.x * scale_log2;
      q[2 * e + 1] = f.y * scale_log2;
    }
  }
  float m = -INFINITY, l = 0.f, o[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i] = 0.f;
  // warp-uniform trip count (the shuffles need every lane); groups past p contribute nothing
  for (int jb = warp * KPW; jb <= p; jb += NG) {
    const int j = jb + grp;
    const bool valid = j <= p;
    const bf16* kr = cache + (static_cast<int64_t>(b) * T + (valid ? j : 0)) * 3 * dl + dl + h * HD + gl * 8;
    const uint4 kv = *reinterpret_cast<const uint4*>(kr);
    const uint4 vv = *reinterpret_cast<const uint4*>(kr + dl);
    const uint32_t kk[4] = {kv.x, kv.y, kv.z, kv.w}, vw[4] = {vv.x, vv.y, vv.z, vv.w};
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = dev::unpack_bf16x2(kk[e]);
      s = fmaf(q[2 * e], f.x, fmaf(q[2 * e + 1], f.y, s));
    }
#pragma unroll
    for (int x = G / 2; x > 0; x >>= 1) s += __shfl_xor_sync(0xffffffffu, s, x);
    if (!valid) continue;
    const float mn = fmaxf(m, s);
    const float corr = dev::ex2_approx(m - mn), e1 = dev::ex2_approx(s - mn);
    l = l * corr + e1;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = dev::unpack_bf16x2(vw[e]);
      o[2 * e] = o[2 * e] * corr + e1 * f.x;
      o[2 * e + 1] = o[2 * e + 1] * corr + e1 * f.y;
    }
    m = mn;
  }
  if (gl == 0) {
    sm_m[gid] = m;
    sm_l[gid] = l;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) sm_o[gid][gl * 8 + i] = o[i];
  __syncthreads();
  if (threadIdx.x < HD) {
    const int c = threadIdx.x;
    float M = -INFINITY;
    for (int g = 0; g < NG; ++g) M = fmaxf(M, sm_m[g]);
    float L = 0.f, acc = 0.f;
    for (int g = 0; g < NG; ++g) {
      if (sm_m[g] == -INFINITY) continue;
      const float f = dev::ex2_approx(sm_m[g] - M);
      L += sm_l[g] * f;
      acc += sm_o[g][c] * f;
    }
    out[static_cast<int64_t>(b) * dl + h * HD + c] = __float2bfloat16(acc / L);
  }
}

// Split-key decode attention (flash-decoding): grid (B * Hl, S), S = the CTA budget of a launch
// (SW_DECODE_CTAS, 320) over the B * Hl heads, at least 2 and at most 8 (one cluster) -- the
// global-merge variant (SW_DECODE_CLUSTER=0) allows DSPLIT with a budget floor of 1. The position is known on the device
// only (CUDA-graph step), so the splits actually used are chosen there: n = min(S, ceil((p + 1) /
// kps)), kps = SW_DECODE_KPS (64), and the CTAs of splits >= n exit at once. Split s of a head
// takes keys [s c, min(p + 1, (s + 1) c)), c = ceil((p + 1) / n); lanes work in groups of G =
// hd / 8 (16-byte loads) and every warp keeps UNR keys' K / V loads in flight before consuming
// them. The split holding key p reads the new k / v from the step's qkv row and writes them into
// the cache (the fused kv_scatter). Each split leaves an unnormalised (m, l, o) partial; the
// split that takes the last ticket of its head's counter merges them and resets the counter.
// Measured: tools/decode_attn_bench.py (graph-timed kernel: 16 fixed splits 12.8 / 16.5 us at
// p = 512 with 32 / 72 heads, ~8.5 / 9.5 with ~4 splits) and tools/ab_decode.sh (LLaMA-7B step,
// same box: batch 1 2.98 -> 2.80 ms/token, batch 8 3.87 -> 3.36).
#ifndef SW_DSPLIT
#define SW_DSPLIT 16
#endif
#ifndef SW_DUNR
#define SW_DUNR 2
#endif
#ifndef SW_DKPS
#define SW_DKPS 64
#endif
#ifndef SW_DCTAS
#define SW_DCTAS 320
#endif
// fewest keys per split (SW_DECODE_KPS) and the CTA budget of one launch (SW_DECODE_CTAS)
int env_or(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e != nullptr && std::atoi(e) > 0 ? std::atoi(e) : dflt;
}
int decode_kps() {
  static const int v = env_or("SW_DECODE_KPS", SW_DKPS);
  return v;
}
int decode_ctas() {
  static const int v = env_or("SW_DECODE_CTAS", SW_DCTAS);
  return v;
}
constexpr int DSPLIT = SW_DSPLIT;  // most splits (partial buffer rows per head)
constexpr int DUNR = SW_DUNR;


// CL: the splits of a head form one thread-block cluster (grid.y = cluster size <= 8) and their
// partials meet in distributed shared memory: split 0 merges them after a cluster barrier, so
// there is no global partial round trip, fence or ticket (SW_DECODE_CLUSTER=0: the global path).
template <int HD, bool CL>
__global__ void __launch_bounds__(256) decode_attention_split_kernel(const bf16* __restrict__ qnew,
                                                                     bf16* __restrict__ cache,
                                                                     bf16* __restrict__ out, int T, int p,
                                                                     const int* __restrict__ pd, int Hl,
                                                                     float scale_log2, float* __restrict__ part,
                                                                     unsigned int* __restrict__ ticket, int kps,
                                                                     int max_split) {
  asm volatile("griddepcontrol.launch_dependents;");  // the output projection may start streaming
  if (pd != nullptr) p = *pd;
  constexpr int G = HD / 8;
  constexpr int KPW = 32 / G;
  constexpr int NG = 8 * KPW;
  __shared__ float sm_m[NG], sm_l[NG];
  __shared__ float sm_o[NG][HD];
  __shared__ bool last;
  __shared__ float sm_part[HD + 2];  // CL: this split's (M, L, unnormalised O)
  const int bh = blockIdx.x, b = bh / Hl, h = bh % Hl, sp = blockIdx.y;
  const int dl = Hl * HD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / G, gl = lane % G;
  const int gid = warp * KPW + grp;
  const int nk = p + 1;
  const int nsplit = max(1, min(max_split, (nk + kps - 1) / kps));
  if (!CL && sp >= nsplit) return;  // a cluster's idle splits still meet its barriers (empty range)
  const int chunk = (nk + nsplit - 1) / nsplit;
  const int k0 = sp < nsplit ? sp * chunk : nk, k1 = sp < nsplit ? min(nk, k0 + chunk) : nk;
  if constexpr (CL) {
    // launched as a programmatic dependent of the QKV GEMM: the cached keys / values (every row
    // but p, which that GEMM is producing) are requested into L2 before waiting for it
    for (int i = threadIdx.x; i < 2 * (k1 - k0) * (HD / 64); i += blockDim.x) {
      const int j = k0 + i / (2 * (HD / 64));
      const int part = i % (2 * (HD / 64));  // K or V, 128-byte line of the head's row
      if (j != p)
        dev::prefetch_l2(cache + (static_cast<int64_t>(b) * T + j) * 3 * dl + dl + (part / (HD / 64)) * dl + h * HD +
                         (part % (HD / 64)) * 64);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  const bf16* qrow = qnew + static_cast<int64_t>(b) * 3 * dl;
  float q[8];
  {
    const uint4 qv = *reinterpret_cast<const uint4*>(qrow + h * HD + gl * 8);
    const uint32_t qq[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = dev::unpack_bf16x2(qq[e]);
      q[2 * e] = f.x * scale_log2;
      q[2 * e + 1] = f.y * scale_log2;
    }
  }
  float m = -INFINITY, l = 0.f, o[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i] = 0.f;
  for (int jb = k0 + warp * KPW; jb < k1; jb += NG * DUNR) {
    uint4 kv[DUNR], vv[DUNR];
#pragma unroll
    for (int u = 0; u < DUNR; ++u) {  // all of this warp's loads first
      const int j = jb + u * NG + grp;
      const int jj = j < k1 ? j : k0;
      const bf16* kr = jj == p ? qrow + dl + h * HD + gl * 8
                               : cache + (static_cast<int64_t>(b) * T + jj) * 3 * dl + dl + h * HD + gl * 8;
      kv[u] = *reinterpret_cast<const uint4*>(kr);
      vv[u] = *reinterpret_cast<const uint4*>(kr + dl);
      if (jj == p && j == p) {  // the new row joins the cache (fused kv_scatter); j past this split's
                                // range (jj = k0) must not write, even when it equals p
        bf16* cr = cache + (static_cast<int64_t>(b) * T + p) * 3 * dl + dl + h * HD + gl * 8;
        *reinterpret_cast<uint4*>(cr) = kv[u];
        *reinterpret_cast<uint4*>(cr + dl) = vv[u];
      }
    }
#pragma unroll
    for (int u = 0; u < DUNR; ++u) {
      const int j = jb + u * NG + grp;
      const uint32_t kk[4] = {kv[u].x, kv[u].y, kv[u].z, kv[u].w}, vw[4] = {vv[u].x, vv[u].y, vv[u].z, vv[u].w};
      float sc = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = dev::unpack_bf16x2(kk[e]);
        sc = fmaf(q[2 * e], f.x, fmaf(q[2 * e + 1], f.y, sc));
      }
#pragma unroll
      for (int x = G / 2; x > 0; x >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, x);
      if (j < k1) {
        const float mn = fmaxf(m, sc);
        const float corr = dev::ex2_approx(m - mn), e1 = dev::ex2_approx(sc - mn);
        l = l * corr + e1;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = dev::unpack_bf16x2(vw[e]);
          o[2 * e] = o[2 * e] * corr + e1 * f.x;
          o[2 * e + 1] = o[2 * e + 1] * corr + e1 * f.y;
        }
        m = mn;
      }
    }
  }
  if (gl == 0) {
    sm_m[gid] = m;
    sm_l[gid] = l;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) sm_o[gid][gl * 8 + i] = o[i];
  __syncthreads();
  float* mine = CL ? sm_part : part + (static_cast<int64_t>(bh) * DSPLIT + sp) * (HD + 2);
  if (threadIdx.x < HD) {  // this split's partial: (M, L, unnormalised O) over its groups
    const int c = threadIdx.x;
    float M = -INFINITY;
    for (int g = 0; g < NG; ++g) M = fmaxf(M, sm_m[g]);
    float L = 0.f, acc = 0.f;
    if (M != -INFINITY) {
      for (int g = 0; g < NG; ++g) {
        if (sm_m[g] == -INFINITY) continue;
        const float f = dev::ex2_approx(sm_m[g] - M);
        L += sm_l[g] * f;
        acc += sm_o[g][c] * f;
      }
    }
    mine[2 + c] = acc;
    if (c == 0) {
      mine[0] = M;
      mine[1] = L;
    }
  }
  if constexpr (CL) {
    dev::cluster_sync();  // every split's partial is in its shared memory
    if (sp == 0 && threadIdx.x < HD) {
      const int c = threadIdx.x;
      const uint32_t base = dev::smem_u32(sm_part);
      float Ms[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) Ms[r] = r < nsplit ? dev::ld_shared_cluster_f32(dev::mapa_shared(base, r)) : -INFINITY;
      float M = -INFINITY;
#pragma unroll
      for (int r = 0; r < 8; ++r) M = fmaxf(M, Ms[r]);
      float L = 0.f, acc = 0.f;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        if (r >= nsplit || Ms[r] == -INFINITY) continue;
        const float f = dev::ex2_approx(Ms[r] - M);
        L += dev::ld_shared_cluster_f32(dev::mapa_shared(base + 4, r)) * f;
        acc += dev::ld_shared_cluster_f32(dev::mapa_shared(base + 4 * (2 + c), r)) * f;
      }
      out[static_cast<int64_t>(b) * dl + h * HD + c] = __float2bfloat16(acc / L);
    }
    dev::cluster_sync();  // the partials have been read
    return;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    last = atomicAdd(ticket + bh, 1u) == static_cast<unsigned>(nsplit - 1);
    if (last) ticket[bh] = 0;  // every split of this head has arrived
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < HD) {
    const int c = threadIdx.x;
    const float* ph = part + static_cast<int64_t>(bh) * DSPLIT * (HD + 2);
    float M = -INFINITY;
    for (int s2 = 0; s2 < nsplit; ++s2) M = fmaxf(M, __ldcg(ph + s2 * (HD + 2)));
    float L = 0.f, acc = 0.f;
    for (int s2 = 0; s2 < nsplit; ++s2) {
      const float ms = __ldcg(ph + s2 * (HD + 2));
      if (ms == -INFINITY) continue;
      const float f = dev::ex2_approx(ms - M);
      L += __ldcg(ph + s2 * (HD + 2) + 1) * f;
      acc += __ldcg(ph + s2 * (HD + 2) + 2 + c) * f;
    }
    out[static_cast<int64_t>(b) * dl + h * HD + c] = __float2bfloat16(acc / L);
  }
}

// Any head dim <= 256 (scalar loads): lane i holds head-dim elements i, i+32, ...
template <int HDV>
__global__ void __launch_bounds__(256) decode_attention_any_kernel(const bf16* __restrict__ qnew,
                                                                   const bf16* __restrict__ cache,
                                                                   bf16* __restrict__ out, int T, int p,
                                                                   const int* __restrict__ pd, int Hl,
                                                                   int hd, float scale_log2) {
  if (pd != nullptr) p = *pd;
  constexpr int WARPS = 8;
  __shared__ float sm_m[WARPS], sm_l[WARPS];
  __shared__ float sm_o[WARPS][32 * HDV];
  const int b = blockIdx.x / Hl, h = blockIdx.x % Hl;
  const int dl = Hl * hd;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float q[HDV];
  const bf16* qr = qnew + static_cast<int64_t>(b) * 3 * dl + h * hd;
#pragma unroll
  for (int i = 0; i < HDV; ++i) {
    const int c = lane + 32 * i;
    q[i] = c < hd ? __bfloat162float(qr[c]) * scale_log2 : 0.f;
  }
  float m = -INFINITY, l = 0.f, o[HDV];
#pragma unroll
  for (int i = 0; i < HDV; ++i) o[i] = 0.f;
  for (int j = warp; j <= p; j += WARPS) {
    const bf16* kr = cache + (static_cast<int64_t>(b) * T + j) * 3 * dl + dl + h * hd;
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < HDV; ++i) {
      const int c = lane + 32 * i;
      if (c < hd) s += q[i] * __bfloat162float(kr[c]);
    }
#pragma unroll
    for (int x = 16; x > 0; x >>= 1) s += __shfl_xor_sync(0xffffffffu, s, x);
    const float mn = fmaxf(m, s);
    const float corr = dev::ex2_approx(m - mn), e = dev::ex2_approx(s - mn);
    l = l * corr + e;
    const bf16* vr = kr + dl;
#pragma unroll
    for (int i = 0; i < HDV; ++i) {
      const int c = lane + 32 * i;
      o[i] = o[i] * corr + (c < hd ? e * __bfloat162float(vr[c]) : 0.f);
    }
    m = mn;
  }
  if (lane == 0) {
    sm_m[warp] = m;
    sm_l[warp] = l;
  }
#pragma unroll
  for (int i = 0; i < HDV; ++i) sm_o[warp][lane + 32 * i] = o[i];
  __syncthreads();
  if (warp == 0) {
    float M = -INFINITY;
    for (int w = 0; w < WARPS; ++w) M = fmaxf(M, sm_m[w]);
    float L = 0.f, acc[HDV];
#pragma unroll
    for (int i = 0; i < HDV; ++i) acc[i] = 0.f;
    for (int w = 0; w < WARPS; ++w) {
      if (sm_m[w] == -INFINITY) continue;
      const float f = dev::ex2_approx(sm_m[w] - M);
      L += sm_l[w] * f;
#pragma unroll
      for (int i = 0; i < HDV; ++i) acc[i] += sm_o[w][lane + 32 * i] * f;
    }
    bf16* orow = out + static_cast<int64_t>(b) * dl + h * hd;
#pragma unroll
    for (int i = 0; i < HDV; ++i) {
      const int c = lane + 32 * i;
      if (c < hd) orow[c] = __float2bfloat16(acc[i] / L);
    }
  }
}

// First maximum of each row (kernels.hpp:515-527 semantics: strict > keeps the lowest index).
// Writes (value, global index) as floats so ranks can combine shards.
// argmax of row b over columns [blockIdx.y * chunk, ...) -> out[(b * gridDim.y + blockIdx.y) * 2 + {0, 1}]
// (value, index_base + column); ties to the smaller index
__global__ void argmax_rows_kernel(const bf16* __restrict__ x, int64_t row_stride, int n, int index_base,
                                   float* __restrict__ out) {
  const int b = blockIdx.x;
  const int chunk = (n + gridDim.y - 1) / gridDim.y;
  const int i0 = blockIdx.y * chunk, i1 = min(n, i0 + chunk);
  const bf16* xr = x + static_cast<int64_t>(b) * row_stride;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const float v = __bfloat162float(xr[i]);
    if (v > best || (v == best && i < bi)) {
      best = v;
      bi = i;
    }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
#pragma unroll
  for (int x2 = 16; x2 > 0; x2 >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, x2);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, x2);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sv[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k) {
      if (sv[k] > best || (sv[k] == best && si[k] < bi)) {
        best = sv[k];
        bi = si[k];
      }
    }
    const int64_t o = (static_cast<int64_t>(b) * gridDim.y + blockIdx.y) * 2;
    out[o] = best;
    out[o + 1] = bi == 0x7fffffff ? -1.f : static_cast<float>(index_base + bi);
  }
}

// parts [B][C][2] -> out [B][2], first maximum (smallest index among equal values)
__global__ void argmax_chunks_kernel(const float* __restrict__ parts, int C, int B, float* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  float best = -INFINITY, bi = -1.f;
  for (int c = 0; c < C; ++c) {
    const float v = parts[(static_cast<int64_t>(b) * C + c) * 2], i = parts[(static_cast<int64_t>(b) * C + c) * 2 + 1];
    if (i < 0.f) continue;
    if (bi < 0.f || v > best || (v == best && i < bi)) {
      best = v;
      bi = i;
    }
  }
  out[2 * b] = best;
  out[2 * b + 1] = bi;
}

// parts[r][b] = (value, index) of shard r; token[b] = index of the first maximum over shards
// (shards hold ascending vocab ranges, so the lowest rank wins ties like the global argmax).
__global__ void argmax_combine_kernel(const float* __restrict__ parts, int shards, int B, int32_t* __restrict__ tok) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  float best = -INFINITY;
  int bi = 0;
  for (int r = 0; r < shards; ++r) {
    const float v = parts[(static_cast<int64_t>(r) * B + b) * 2];
    if (v > best) {
      best = v;
      bi = static_cast<int>(parts[(static_cast<int64_t>(r) * B + b) * 2 + 1]);
    }
  }
  tok[b] = bi;
}

}  // namespace

void embed_rows(const int32_t* ids, const float* tok, const float* pos, int p, float* x, int B, int d, cudaStream_t s,
                const int* p_dev) {
  embed_rows_kernel<<<B, 256, 0, s>>>(ids, tok, pos, p, p_dev, x, d);
}

void kv_scatter(const bf16* qkv_new, bf16* cache, int B, int T, int p, int dl, cudaStream_t s, const int* p_dev) {
  kv_scatter_kernel<<<B, 128, 0, s>>>(qkv_new, cache, T, p, p_dev, dl);
}

void decode_attention(const bf16* qkv_new, const bf16* cache, bf16* out, int B, int T, int p, int Hl, int hd,
                      cudaStream_t s, const int* p_dev) {
  const float scale_log2 = static_cast<float>(1.4426950408889634 / sqrt(static_cast<double>(hd)));
  switch (hd) {
    case 64: decode_attention_kernel<64><<<B * Hl, 256, 0, s>>>(qkv_new, cache, out, T, p, p_dev, Hl, scale_log2); break;
    case 128: decode_attention_kernel<128><<<B * Hl, 256, 0, s>>>(qkv_new, cache, out, T, p, p_dev, Hl, scale_log2); break;
    case 256: decode_attention_kernel<256><<<B * Hl, 256, 0, s>>>(qkv_new, cache, out, T, p, p_dev, Hl, scale_log2); break;
    default:
      if (hd > 256) throw std::runtime_error("decode_attention: head_dim must be <= 256");
      if (hd <= 64) {
        decode_attention_any_kernel<2><<<B * Hl, 256, 0, s>>>(qkv_new, cache, out, T, p, p_dev, Hl, hd, scale_log2);
      } else if (hd <= 128) {
        decode_attention_any_kernel<4><<<B * Hl, 256, 0, s>>>(qkv_new, cache, out, T, p, p_dev, Hl, hd, scale_log2);
      } else {
        decode_attention_any_kernel<8><<<B * Hl, 256, 0, s>>>(qkv_new, cache, out, T, p, p_dev, Hl, hd, scale_log2);
      }
  }
}

__global__ void bump_kernel(int* x) { *x += 1; }

void bump_i32(int* x, cudaStream_t s) { bump_kernel<<<1, 1, 0, s>>>(x); }

// SW_DECODE_PDL=0: the decode attention / LayerNorm kernels wait for their predecessor to finish
bool decode_pdl_on() {
  static const bool on = [] {
    const char* e = std::getenv("SW_DECODE_PDL");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

bool decode_cluster_on() {
  static const bool on = [] {
    const char* e = std::getenv("SW_DECODE_CLUSTER");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

template <int HD>
void launch_decode_split(const bf16* qkv_new, bf16* cache, bf16* out, int B, int T, int p, int Hl, float scale_log2,
                         cudaStream_t s, const int* p_dev, float* part, unsigned int* ticket) {
  const int kps = decode_kps();
  if (decode_cluster_on()) {
    // splits per head: keys / kps, at most the CTA budget over the B * Hl heads and the portable
    // cluster size
    // (at least two: with many heads one split per head leaves each CTA the whole context)
    const int max_split = std::max(2, std::min(8, decode_ctas() / (B * Hl)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(B * Hl), static_cast<unsigned>(max_split));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = static_cast<unsigned>(max_split);
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = decode_pdl_on() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, decode_attention_split_kernel<HD, true>, qkv_new, cache, out, T,
                                             p, p_dev, Hl, scale_log2, part, ticket, kps, max_split);
    if (e != cudaSuccess) throw std::runtime_error(std::string("decode attention launch: ") + cudaGetErrorString(e));
    return;
  }
  const int max_split = std::max(1, std::min(DSPLIT, decode_ctas() / (B * Hl)));
  const dim3 grid(B * Hl, max_split);
  decode_attention_split_kernel<HD, false><<<grid, 256, 0, s>>>(qkv_new, cache, out, T, p, p_dev, Hl, scale_log2,
                                                                part, ticket, kps, max_split);
}

bool decode_attention_split(const bf16* qkv_new, bf16* cache, bf16* out, int B, int T, int p, int Hl, int hd,
                            cudaStream_t s, const int* p_dev, float* part, unsigned int* ticket) {
  const float scale_log2 = static_cast<float>(1.4426950408889634 / sqrt(static_cast<double>(hd)));
  switch (hd) {
    case 64:
      launch_decode_split<64>(qkv_new, cache, out, B, T, p, Hl, scale_log2, s, p_dev, part, ticket);
      return true;
    case 128:
      launch_decode_split<128>(qkv_new, cache, out, B, T, p, Hl, scale_log2, s, p_dev, part, ticket);
      return true;
    case 256:
      launch_decode_split<256>(qkv_new, cache, out, B, T, p, Hl, scale_log2, s, p_dev, part, ticket);
      return true;
    default:
      return false;
  }
}

int decode_split_count() { return DSPLIT; }

void argmax_rows(const bf16* x, int64_t row_stride, int B, int n, int index_base, float* out, cudaStream_t s,
                 float* scratch) {
  // one CTA per row is a single SM streaming the whole vocabulary row: with scratch, the row is
  // cut into up to 64 chunks of >= 1024 columns and the chunk winners are combined
  const int C = scratch != nullptr ? std::max(1, std::min(kArgmaxChunks, n / 1024)) : 1;
  if (C == 1) {
    argmax_rows_kernel<<<dim3(B, 1), 256, 0, s>>>(x, row_stride, n, index_base, out);
    return;
  }
  argmax_rows_kernel<<<dim3(B, C), 256, 0, s>>>(x, row_stride, n, index_base, scratch);
  argmax_chunks_kernel<<<(B + 127) / 128, 128, 0, s>>>(scratch, C, B, out);
}

void argmax_combine(const float* parts, int shards, int B, int32_t* tok, cudaStream_t s) {
  argmax_combine_kernel<<<(B + 127) / 128, 128, 0, s>>>(parts, shards, B, tok);
}

}  // namespace k
}  // namespace sw
