// Host-side interface of the tcgen05 GEMM family.
//
// Logical product: C[M, N] = sum_k A[m, k] * B[n, k]   (bf16 operands, fp32 accumulation in TMEM)
//
// Each operand is either K-major (row r at ptr + r*ld, k contiguous) or MN-major
// (k-th row at ptr + k*ld, m/n contiguous). With weights stored [out, in] (graph.hpp:353-375)
// the three linear-layer products are
//   forward   y  = x . W^T   : A = x  (K-major),  B = W   (K-major)
//   dgrad     dx = dy . W    : A = dy (K-major),  B = W   (MN-major)
//   wgrad     dW = dy^T . x  : A = dy (MN-major), B = x   (MN-major)
// so no operand is ever transposed in memory.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sw {

enum class Epi : int {
  kStoreBf16 = 0,   // C(bf16) = alpha*acc (+ bias)
  kStoreF32 = 1,    // C(f32)  = alpha*acc (+ bias) (+ C if accumulate)
  kBiasGelu = 2,    // C(bf16) = acc + bias (pre-activation), C2(bf16) = gelu(acc + bias)
  kResidF32 = 3,    // C(f32)  = aux(f32) + acc + bias     (residual stream update; C may alias aux)
  kGeluBwd = 4,     // C(bf16) = acc * gelu'(aux(bf16))    (fc2 dgrad fused with GeLU backward)
  kAdamW = 5,       // wgrad with the optimizer in the epilogue: acc is the fp32 gradient of the
                    // [M, N] weight at adam_* (row pitch ldc); AdamW updates p/m/v in place and
                    // refreshes the bf16 shadow; non-finite gradients set *adam_flag, and a
                    // non-zero *adam_flag on entry to a chunk gates its update (state unchanged)
  // SwiGLU extension. kSwiGLU: B = fused [gate; up] weight [2*N, K] (up rows start at
  // swiglu_half = N); each 256-wide tile multiplies 128 gate rows and the matching 128 up rows,
  // the epilogue writes h = silu(g) * u to C [M, N] and the pre-activations g | u to C2 [M, 2N].
  // kSwiGLUBwd: acc = dh [M, N]; aux = g | u [M, 2N]; C [M, 2N] = dh*u*silu'(g) | dh*silu(g).
  kSwiGLU = 6,
  kSwiGLUBwd = 7,
  // kBf16Delta: the attention-output gradient GEMM with the flash-attention backward's row
  // statistic fused in: C(bf16) = alpha*acc and, per row r = b*delta_T + t and 128-column head h,
  // delta[(b*(N/128) + h)*delta_T + t] = sum_c bf16(C[r, c]) * aux(bf16)[r, c] (aux = the forward
  // attention output O). CTA-pair TMA-store path only (gemm_delta_ok).
  kBf16Delta = 8,
};

struct GemmParams {
  int M = 0, N = 0, K = 0;
  const void* A = nullptr;
  int64_t lda = 0;
  int a_mn_major = 0;
  const void* B = nullptr;
  int64_t ldb = 0;
  int b_mn_major = 0;
  Epi epi = Epi::kStoreBf16;
  void* C = nullptr;
  int64_t ldc = 0;
  void* C2 = nullptr;
  int64_t ldc2 = 0;
  const float* bias = nullptr;
  // Segmented bias: column n reads bias[(n / bias_seg) * bias_seg_stride + n % bias_seg]
  // (fused QKV: three column blocks whose biases live in three separate full-width vectors).
  int bias_seg = 0;  // 0 = plain bias[n]
  int64_t bias_seg_stride = 0;
  const void* aux = nullptr;
  int64_t ld_aux = 0;
  int swiglu_half = 0;  // kSwiGLU / kSwiGLUBwd: N of the h activations (row offset of up in B)
  float alpha = 1.0f;
  int accumulate = 0;
  // kAdamW (train_state.hpp:211-216, Scalar = float)
  float* adam_p = nullptr;
  float* adam_m = nullptr;
  float* adam_v = nullptr;
  void* adam_w = nullptr;
  int* adam_flag = nullptr;
  float adam_lr = 0.f, adam_b1 = 0.f, adam_b2 = 0.f, adam_eps = 0.f, adam_wd = 0.f, adam_c1 = 1.f, adam_c2 = 1.f;
  int adam_fast = 0;  // set by gemm_bf16: bias corrections in [2^-14, 1] admit the branch-free path
  int num_sms = 0;  // 0 = all
  int trace_cta = -1;  // profiling: CTA whose per-tile phases are stamped (SW_GEMM_TRACE_CTA)
  float* delta = nullptr;  // kBf16Delta output [M / delta_T][N / 128][delta_T]
  // kGeluBwd: per-32-row partial column sums of the stored bf16 output, [ceil(M / 32)][N] (the
  // bias gradient of the GeLU layer; reduce with k::colsum_chunks). Requires gemm_colsum_ok.
  float* colsum = nullptr;
  int delta_T = 0;
  // ReLU instead of GeLU (T5 MLP): kStoreBf16 stores relu(acc + bias); kGeluBwd multiplies by
  // relu'(aux) = (aux > 0) with aux = the stored ReLU output
  int relu = 0;
  // Decode: launch the weight-streaming kernel as a programmatic dependent of the previous kernel
  // in the stream (its first weight lines are requested before griddepcontrol.wait)
  int pdl = 0;
  // kStoreF32 only: K split into this many slices whose fp32 partial tiles are reduce-added into C
  // by TMA (0 = chosen by gemm_bf16 for GEMMs with too few tiles to fill the GPU; C is zeroed
  // first unless accumulate). Summation order differs from the unsplit GEMM (fp32 rounding).
  int split_k = 0;
};

// Returns cudaSuccess or the launch error. Throws std::runtime_error on invalid shapes.
cudaError_t gemm_bf16(const GemmParams& p, cudaStream_t stream);

// Whether gemm_bf16 can run p with epi = kBf16Delta (CTA-pair kernel with the TMA-store epilogue,
// 128-column heads, no accumulate, M a multiple of delta_T).
bool gemm_delta_ok(const GemmParams& p);
// Whether a kGeluBwd call can also write the partial column sums (p.colsum).
bool gemm_colsum_ok(const GemmParams& p);

// The split-K slice count gemm_bf16 would use for p run as an fp32-store GEMM (1 = no split).
int gemm_split_k(const GemmParams& p);

// Profiling: the 1024 per-tile phase stamps of the CTA named by SW_GEMM_TRACE_CTA.
void gemm_trace_read(unsigned long long* out);

}  // namespace sw
