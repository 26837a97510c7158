// tcgen05.mma issue-rate microbenchmark: cycles per kind::f16 MMA (K = 16) for the shapes the
// attention kernels use, operands from shared memory (SS) or A from TMEM (TS), one CTA per SM.
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -Ipaper_2310_16355_b200/csrc
//        tools/mma_micro.cu -o tools/mma_micro
// Shared memory content is garbage: only timing matters.
#include <cstdio>
#include <cstdint>

#include "sm100.cuh"

using namespace sw;

template <int M, int N, int MODE>  // MODE 0: SS K-major A/B; 1: SS, B MN-major; 2: TS (A in TMEM); 3: SS, A and B MN-major
__global__ void __launch_bounds__(128, 1) mma_rate(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 200 * 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const uint32_t warp = dev::warp_idx_sync();
  if (threadIdx.x == 0) {
    dev::mbar_init(bar, 1);
    dev::fence_barrier_init();
  }
  if (warp == 0) dev::tmem_alloc<512>(slot);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 1) {
    const uint32_t idesc = dev::make_idesc_bf16(M, N, MODE == 3 ? 1 : 0, (MODE == 1 || MODE == 3) ? 1 : 0);
    const uint64_t da = dev::make_sdesc_sw128(dev::smem_u32(smem), MODE == 3 ? 8192 : 16, 1024);
    const uint64_t db = dev::make_sdesc_sw128(dev::smem_u32(smem + 64 * 1024), (MODE == 1 || MODE == 3) ? 8192 : 16, 1024);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (dev::elect_one_sync()) {
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
          if (MODE == 2)
            dev::umma_f16_ts(tmem + 256, tmem + (kk & 7) * 8, db + ((kk & 3) * 2), idesc, 1u);
          else if (MODE == 3)
            dev::umma_f16_ss(tmem, da + ((kk & 3) * 128), db + ((kk & 3) * 128), idesc, 1u);
          else if (MODE == 1)
            dev::umma_f16_ss(tmem, da + ((kk & 3) * 2), db + ((kk & 3) * 128), idesc, 1u);
          else
            dev::umma_f16_ss(tmem, da + ((kk & 3) * 2), db + ((kk & 3) * 2), idesc, 1u);
        }
      }
      __syncwarp();
    }
    if (dev::elect_one_sync()) dev::umma_commit(bar);
    __syncwarp();
    dev::mbar_wait(bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 32 && blockIdx.x == 0) out[0] = static_cast<unsigned long long>(t1 - t0);
  }
  dev::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    dev::tc_fence_after();
    dev::tmem_dealloc<512>(tmem);
  }
}

template <int M, int N, int MODE>
void run(const char* name, unsigned long long* d_out) {
  const int iters = 256;
  cudaFuncSetAttribute(mma_rate<M, N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 201 * 1024);
  for (int rep = 0; rep < 2; ++rep) mma_rate<M, N, MODE><<<148, 128, 201 * 1024>>>(d_out, iters);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long cyc = 0;
  cudaMemcpy(&cyc, d_out, 8, cudaMemcpyDeviceToHost);
  const double per = static_cast<double>(cyc) / (iters * 16.0);
  const double floor = (M < 128 ? 128 : M) * N / 256.0;
  printf("{\"shape\": \"%s\", \"cycles_per_mma\": %.1f, \"floor\": %.0f, \"err\": \"%s\"}\n", name, per, floor,
         cudaGetErrorString(e));
}

int main() {
  unsigned long long* d_out;
  cudaMalloc(&d_out, 64);
  run<128, 64, 0>("SS M128 N64 K-major", d_out);
  run<128, 64, 1>("SS M128 N64 B MN-major", d_out);
  run<128, 128, 0>("SS M128 N128 K-major", d_out);
  run<128, 128, 1>("SS M128 N128 B MN-major", d_out);
  run<128, 256, 0>("SS M128 N256 K-major", d_out);
  run<128, 256, 1>("SS M128 N256 B MN-major", d_out);
  run<128, 256, 3>("SS M128 N256 A+B MN-major", d_out);
  run<128, 128, 3>("SS M128 N128 A+B MN-major", d_out);
  run<128, 64, 2>("TS M128 N64", d_out);
  run<128, 128, 2>("TS M128 N128", d_out);
  return 0;
}
