// Checks the branch-free division / square root of sm100.cuh (div_rn_fast, sqrt_rn_fast) against
// the compiler's IEEE __fdiv_rn / __fsqrt_rn: exhaustively over every float for sqrt, and over
// 2^32 x 4 structured-random operand pairs for division. Wherever the fast path reports ok, the
// bits must be identical. Also reports how much of the range is accepted.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -Ipaper_2310_16355_b200/csrc \
//        tools/verify_fastmath.cu -o /tmp/verify_fastmath
#include <cstdio>
#include <cstdint>

#include "sm100.cuh"

__device__ unsigned long long g_bad_sqrt, g_ok_sqrt, g_bad_div, g_ok_div;

__global__ void sqrt_all(uint64_t base) {
  const uint64_t i = base + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i > 0xffffffffull) return;
  const float x = __uint_as_float(static_cast<uint32_t>(i));
  bool ok = true;
  const float f = sw::dev::sqrt_rn_fast(x, ok);
  const float e = __fsqrt_rn(x);
  if (ok) {
    atomicAdd(&g_ok_sqrt, 1ull);
    if (__float_as_uint(f) != __float_as_uint(e)) atomicAdd(&g_bad_sqrt, 1ull);
  }
}

__device__ __forceinline__ uint32_t hash32(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return static_cast<uint32_t>(z ^ (z >> 31));
}

__global__ void div_random(uint64_t base, int mode) {
  const uint64_t i = base + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  uint32_t ua = hash32(2 * i + 17 * mode), ub = hash32(2 * i + 1 + 17 * mode);
  if (mode == 1) ub = (ub & 0x807fffffu) | ((96u + (ub >> 24) % 64u) << 23);        // b near 1 (like c1, c2)
  if (mode == 2) ua = (ua & 0x807fffffu) | ((20u + (ua >> 24) % 140u) << 23);       // small a (m, v)
  if (mode == 3) ub = (ub & 0x807fffffu) | ((90u + (ub >> 24) % 50u) << 23);        // b ~ sqrt(v)+eps
  if (mode == 4) {                                                                   // a/c, c in (2^-14, 1]
    ub = 0x3f800000u - (ub % 0x07000000u);
  }
  const float a = __uint_as_float(ua), b = __uint_as_float(ub);
  bool ok = true;
  float f;
  if (mode == 4) {
    ok = b >= 1.0f / 16384.0f;
    f = sw::dev::div_rn_fast_c(a, b, sw::dev::rcp_refined(b), ok);
  } else {
    f = sw::dev::div_rn_fast(a, b, ok);
  }
  const float e = __fdiv_rn(a, b);
  if (ok) {
    atomicAdd(&g_ok_div, 1ull);
    if (__float_as_uint(f) != __float_as_uint(e) && !(f == 0.0f && e == 0.0f)) atomicAdd(&g_bad_div, 1ull);
  }
}

int main() {
  const int T = 256;
  for (uint64_t base = 0; base <= 0xffffffffull; base += (1ull << 30)) sqrt_all<<<(1u << 30) / T, T>>>(base);
  for (int mode = 0; mode < 5; ++mode)
    for (uint64_t base = 0; base < (1ull << 32); base += (1ull << 30)) div_random<<<(1u << 30) / T, T>>>(base, mode);
  cudaError_t err = cudaDeviceSynchronize();
  unsigned long long bs, os, bd, od;
  cudaMemcpyFromSymbol(&bs, g_bad_sqrt, 8);
  cudaMemcpyFromSymbol(&os, g_ok_sqrt, 8);
  cudaMemcpyFromSymbol(&bd, g_bad_div, 8);
  cudaMemcpyFromSymbol(&od, g_ok_div, 8);
  std::printf("{\"cuda\": \"%s\", \"sqrt_checked\": %llu, \"sqrt_mismatch\": %llu, \"div_checked\": %llu, "
              "\"div_mismatch\": %llu}\n", cudaGetErrorString(err), os, bs, od, bd);
  return (err == cudaSuccess && bs == 0 && bd == 0) ? 0 : 1;
}
