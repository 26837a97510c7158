// Kernel-level C ABI entry points + the common error/version plumbing.
#include <cstdlib>
#include <string>

#include "gemm.h"
#include "status.h"

namespace sw {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

}  // namespace sw

extern "C" {

const char* sw_last_error(void) { return sw::g_last_error.c_str(); }

const char* sw_version(void) { return "shardweave_b200 0.1 (sm_100a)"; }

void sw_free(void* p) { std::free(p); }

sw_status sw_k_gemm_bf16(int M, int N, int K, const void* A, int64_t lda, int a_mn_major,
                         const void* B, int64_t ldb, int b_mn_major, int epi, void* C, int64_t ldc,
                         void* C2, int64_t ldc2, const float* bias, const void* aux,
                         int64_t ld_aux, float alpha, int accumulate, void* stream) {
  return sw::guarded([&] {
    if (epi < 0 || epi > 4) sw::fail(SW_ERR_CONFIG, "sw_k_gemm_bf16: unknown epilogue");
    sw::GemmParams p;
    p.M = M;
    p.N = N;
    p.K = K;
    p.A = A;
    p.lda = lda;
    p.a_mn_major = a_mn_major;
    p.B = B;
    p.ldb = ldb;
    p.b_mn_major = b_mn_major;
    p.epi = static_cast<sw::Epi>(epi);
    p.C = C;
    p.ldc = ldc;
    p.C2 = C2;
    p.ldc2 = ldc2;
    p.bias = bias;
    p.aux = aux;
    p.ld_aux = ld_aux;
    p.alpha = alpha;
    p.accumulate = accumulate;
    sw::cuda_check(sw::gemm_bf16(p, static_cast<cudaStream_t>(stream)), "gemm_bf16 launch");
  });
}

}  // extern "C"
