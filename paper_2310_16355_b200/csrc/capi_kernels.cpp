// Kernel-level C ABI entry points + the common error/version plumbing.
#include <cstdlib>
#include <string>

#include "gemm.h"
#include "kernels.h"
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
    if ((epi < 0 || epi > 4) && epi != 8) sw::fail(SW_ERR_CONFIG, "sw_k_gemm_bf16: unknown epilogue");
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
    if (p.epi == sw::Epi::kBf16Delta) {  // C2 carries the fp32 delta output, ldc2 the sequence length
      p.delta = static_cast<float*>(C2);
      p.delta_T = static_cast<int>(ldc2);
      p.C2 = nullptr;
      p.ldc2 = 0;
      if (!sw::gemm_delta_ok(p)) sw::fail(SW_ERR_CONFIG, "sw_k_gemm_bf16: fused delta not available for this shape");
    }
    sw::cuda_check(sw::gemm_bf16(p, static_cast<cudaStream_t>(stream)), "gemm_bf16 launch");
  });
}

sw_status sw_k_gemm_bf16_swiglu(int M, int N, int K, const void* A, int64_t lda, const void* W_gu, int64_t ldw,
                                void* h, int64_t ldh, void* pre, int64_t ldpre, void* stream) {
  return sw::guarded([&] {
    sw::GemmParams g;
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = A;
    g.lda = lda;
    g.B = W_gu;
    g.ldb = ldw;
    g.epi = sw::Epi::kSwiGLU;
    g.C = h;
    g.ldc = ldh;
    g.C2 = pre;
    g.ldc2 = ldpre;
    g.swiglu_half = N;
    sw::cuda_check(sw::gemm_bf16(g, static_cast<cudaStream_t>(stream)), "gemm_bf16_swiglu launch");
  });
}

sw_status sw_k_gemm_bf16_swiglu_bwd(int M, int N, int K, const void* A, int64_t lda, int a_mn_major, const void* B,
                                    int64_t ldb, int b_mn_major, const void* pre, int64_t ldpre, void* dpre,
                                    int64_t lddpre, void* stream) {
  return sw::guarded([&] {
    sw::GemmParams g;
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = A;
    g.lda = lda;
    g.a_mn_major = a_mn_major;
    g.B = B;
    g.ldb = ldb;
    g.b_mn_major = b_mn_major;
    g.epi = sw::Epi::kSwiGLUBwd;
    g.C = dpre;
    g.ldc = lddpre;
    g.aux = pre;
    g.ld_aux = ldpre;
    g.swiglu_half = N;
    sw::cuda_check(sw::gemm_bf16(g, static_cast<cudaStream_t>(stream)), "gemm_bf16_swiglu_bwd launch");
  });
}

sw_status sw_k_gemm_bf16_adamw(int M, int N, int K, const void* A, int64_t lda, int a_mn_major, const void* B,
                               int64_t ldb, int b_mn_major, float* p, float* m, float* v, void* shadow, int64_t ld,
                               int* nonfinite_flag, float lr, float b1, float b2, float eps, float wd, float c1,
                               float c2, void* stream) {
  return sw::guarded([&] {
    if (N % 4 != 0 || ld % 4 != 0) sw::fail(SW_ERR_SHAPE, "sw_k_gemm_bf16_adamw: N and ld must be multiples of 4");
    sw::GemmParams g;
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = A;
    g.lda = lda;
    g.a_mn_major = a_mn_major;
    g.B = B;
    g.ldb = ldb;
    g.b_mn_major = b_mn_major;
    g.epi = sw::Epi::kAdamW;
    g.ldc = ld;
    g.adam_p = p;
    g.adam_m = m;
    g.adam_v = v;
    g.adam_w = shadow;
    g.adam_flag = nonfinite_flag;
    g.adam_lr = lr;
    g.adam_b1 = b1;
    g.adam_b2 = b2;
    g.adam_eps = eps;
    g.adam_wd = wd;
    g.adam_c1 = c1;
    g.adam_c2 = c2;
    sw::cuda_check(sw::gemm_bf16(g, static_cast<cudaStream_t>(stream)), "gemm_bf16_adamw launch");
  });
}

sw_status sw_k_decode_attention(const void* qkv_new, void* cache, void* out, int B, int T, int p, int Hl, int hd,
                                int split, float* part, unsigned int* ticket, void* stream) {
  return sw::guarded([&] {
    const auto* q = static_cast<const sw::k::bf16*>(qkv_new);
    auto* c = static_cast<sw::k::bf16*>(cache);
    auto* o = static_cast<sw::k::bf16*>(out);
    const auto st = static_cast<cudaStream_t>(stream);
    if (!(split && sw::k::decode_attention_split(q, c, o, B, T, p, Hl, hd, st, nullptr, part, ticket))) {
      sw::k::kv_scatter(q, c, B, T, p, Hl * hd, st);
      sw::k::decode_attention(q, c, o, B, T, p, Hl, hd, st);
    }
    sw::cuda_check(cudaGetLastError(), "decode_attention");
  });
}

sw_status sw_k_attention_fwd(const void* qkv, void* o, float* lse, int B, int T, int Hl, int hd,
                             void* stream) {
  return sw::guarded([&] {
    sw::k::attention_fwd(static_cast<const sw::k::bf16*>(qkv), static_cast<sw::k::bf16*>(o), lse, B, T, Hl,
                         hd, static_cast<cudaStream_t>(stream));
    sw::cuda_check(cudaGetLastError(), "attention_fwd");
  });
}

sw_status sw_k_attention_bwd(const void* qkv, const void* o, const float* lse, const void* dout,
                             void* dqkv, float* scratch, int B, int T, int Hl, int hd, void* stream) {
  return sw::guarded([&] {
    sw::k::attention_bwd(static_cast<const sw::k::bf16*>(qkv), static_cast<const sw::k::bf16*>(o), lse,
                         static_cast<const sw::k::bf16*>(dout), static_cast<sw::k::bf16*>(dqkv), scratch, B, T,
                         Hl, hd, static_cast<cudaStream_t>(stream));
    sw::cuda_check(cudaGetLastError(), "attention_bwd");
  });
}

long long sw_k_attention_bwd_scratch(int B, int T, int Hl, int hd) {
  return static_cast<long long>(sw::k::attention_bwd_scratch_floats(B, T, Hl, hd));
}

sw_status sw_k_gemm_trace(unsigned long long* out) {
  return sw::guarded([&] { sw::gemm_trace_read(out); });
}

// Debug: clock64 stamps of the traced attention-backward CTA (SW_ATTN_TRACE_CTA), 4096 slots.
sw_status sw_k_attention_trace(unsigned long long* out) {
  return sw::guarded([&] { sw::k::attention_trace_read(out); });
}

sw_status sw_k_layernorm_fwd(const float* x, const float* scale, const float* bias, void* y, float* mean,
                             float* rstd, int64_t M, int d, float eps, void* stream) {
  return sw::guarded([&] {
    sw::k::layernorm_fwd(x, scale, bias, static_cast<sw::k::bf16*>(y), mean, rstd, M, d, eps,
                         static_cast<cudaStream_t>(stream));
    sw::cuda_check(cudaGetLastError(), "layernorm_fwd");
  });
}

sw_status sw_k_layernorm_bwd(const float* x, const float* mean, const float* rstd, const float* scale,
                             const float* dy, float* g_io, void* g_bf16, float* dscale, float* dbias,
                             int64_t M, int d, int accumulate, void* stream) {
  return sw::guarded([&] {
    sw::k::layernorm_bwd(x, mean, rstd, scale, dy, g_io, static_cast<sw::k::bf16*>(g_bf16), dscale, dbias, M,
                         d, accumulate, static_cast<cudaStream_t>(stream));
    sw::cuda_check(cudaGetLastError(), "layernorm_bwd");
  });
}

sw_status sw_k_rmsnorm_fwd(const float* x, const float* scale, void* y, float* rstd, int64_t M, int d, float eps,
                           void* stream) {
  return sw::guarded([&] {
    sw::k::layernorm_fwd(x, scale, nullptr, static_cast<sw::k::bf16*>(y), nullptr, rstd, M, d, eps,
                         static_cast<cudaStream_t>(stream), 1);
    sw::cuda_check(cudaGetLastError(), "rmsnorm_fwd");
  });
}

sw_status sw_k_rmsnorm_bwd(const float* x, const float* rstd, const float* scale, const float* dy, float* g_io,
                           void* g_bf16, float* dscale, int64_t M, int d, int accumulate, void* stream) {
  return sw::guarded([&] {
    sw::k::layernorm_bwd(x, nullptr, rstd, scale, dy, g_io, static_cast<sw::k::bf16*>(g_bf16), dscale, nullptr, M,
                         d, accumulate, static_cast<cudaStream_t>(stream), nullptr, 1);
    sw::cuda_check(cudaGetLastError(), "rmsnorm_bwd");
  });
}

sw_status sw_k_xent(void* logits, int64_t ld, int64_t M, int V, const int32_t* targets, const float* weights,
                    const float* wsum, float* wloss, int write_grad, void* stream) {
  return sw::guarded([&] {
    sw::k::xent_fwd_bwd(static_cast<sw::k::bf16*>(logits), ld, M, V, targets, weights, wsum, wloss, write_grad,
                        static_cast<cudaStream_t>(stream));
    sw::cuda_check(cudaGetLastError(), "xent");
  });
}

sw_status sw_k_adamw(float* p, float* m, float* v, const float* g, void* shadow, int64_t n, float lr,
                     float b1, float b2, float eps, float wd, float c1, float c2, void* stream) {
  return sw::guarded([&] {
    sw::k::adamw(p, m, v, g, static_cast<sw::k::bf16*>(shadow), n, lr, b1, b2, eps, wd, c1, c2,
                 static_cast<cudaStream_t>(stream));
    sw::cuda_check(cudaGetLastError(), "adamw");
  });
}

}  // extern "C"
