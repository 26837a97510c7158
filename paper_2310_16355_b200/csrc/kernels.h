// Launchers of the non-GEMM kernels of the step (HBM-bound elementwise / reduction work).
// Every launcher enqueues exactly one kernel on `s` and returns nothing; errors surface through
// cudaGetLastError at the executor's checkpoints.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace sw {
namespace k {

using bf16 = __nv_bfloat16;

// h[m, :] = tok[ids[m], :] + pos[m % T, :]                       (model.hpp:90-98)
void embed_fwd(const int32_t* ids, const float* tok, const float* pos, float* h, int64_t M, int T,
               int d, cudaStream_t s);
// dtok[ids[m], :] += g[m, :] (atomic); dpos[t, :] (+)= sum_b g[b*T + t, :]   (kernels.hpp:291-304)
// dtok[ids[m]] += g[m] for every position. With `keys` scratch (ceil_pow2(M) uint32) and
// V <= 65535, M <= 65536 the positions are sorted by token (one-CTA bitonic sort) and each token's
// rows are summed in ascending position order (M <= 32768): deterministic, so replicated embedding tables stay
// bit-identical across tensor-parallel ranks like the reference's. keys == nullptr: atomics.
void embed_bwd_tok(const int32_t* ids, const float* g, float* dtok, int64_t M, int d, int V, uint32_t* keys,
                   cudaStream_t s);
int64_t embed_bwd_keys(int64_t M);  // scratch elements embed_bwd_tok needs
void embed_bwd_pos(const float* g, float* dpos, int B, int T, int d, int accumulate, cudaStream_t s);

// LayerNorm over the last dim, biased variance, eps (kernels.hpp:184-215): y = xhat*scale+bias
// (bf16), mean/rstd saved for the backward.
// rms = 1: RMSNorm (extension): no centring, no bias (bias may be null), mean = 0.
void layernorm_fwd(const float* x, const float* scale, const float* bias, bf16* y, float* mean,
                   float* rstd, int64_t M, int d, float eps, cudaStream_t s, int rms = 0);
// Decode-step variant (M <= 8): one-pass statistics, one CTA of 1024 threads per row; other
// sizes fall through to layernorm_fwd.
void layernorm_fwd_small(const float* x, const float* scale, const float* bias, bf16* y, float* mean, float* rstd,
                         int64_t M, int d, float eps, cudaStream_t s, int rms);
// dx = rstd*(g - mean(g) - xhat*mean(g*xhat)), g = dy*scale (kernels.hpp:232-271).
// g_io: residual-stream gradient; g_io = (accumulate ? g_io : 0) + dx; g_bf16 = bf16(g_io).
// dscale += sum_rows dy*xhat, dbias += sum_rows dy (atomics; caller zeroes when needed).
// dscale / dbias: with `partials` scratch (layernorm_bwd_partials(d) floats) every CTA writes its
// column partials and one fixed-order pass adds them (deterministic); partials == nullptr: atomics.
void layernorm_bwd(const float* x, const float* mean, const float* rstd, const float* scale,
                   const float* dy, float* g_io, bf16* g_bf16, float* dscale, float* dbias,
                   int64_t M, int d, int accumulate, cudaStream_t s, float* partials = nullptr, int rms = 0,
                   float* gsum = nullptr);  // gsum: += column sums of the written g_io
// Same, with the residual-stream gradient dy in bf16 (after a bf16 all-reduce).
void layernorm_bwd(const float* x, const float* mean, const float* rstd, const float* scale,
                   const bf16* dy, float* g_io, bf16* g_bf16, float* dscale, float* dbias,
                   int64_t M, int d, int accumulate, cudaStream_t s, float* partials = nullptr, int rms = 0,
                   float* gsum = nullptr);  // gsum: += column sums of the written g_io
int64_t layernorm_bwd_partials(int d);

// Column sums of X [M, N] (bf16 or f32, row pitch ld) written (accumulate=0) or added into
// out: column n goes to outs[n / seg][n % seg] (up to 3 segments). scratch: >= 64*N floats.
void colsum_bf16(const bf16* X, int64_t ld, int64_t M, int N, int seg, float* out0, float* out1,
                 float* out2, int accumulate, float* scratch, cudaStream_t s);
// out[n] (+)= sum_c partial[c * N + n] over `chunks` rows of partial sums, fixed order.
// seg > 0: columns [i*seg, (i+1)*seg) go to out_i (i < 3), like colsum_bf16.
void colsum_chunks(const float* partial, int chunks, int N, float* out, int accumulate, cudaStream_t s,
                   int seg = 0, float* out1 = nullptr, float* out2 = nullptr);
void colsum_f32(const float* X, int64_t ld, int64_t M, int N, float* out, int accumulate,
                float* scratch, cudaStream_t s);

// sum of weights -> wsum[0]
// Greedy decode (decode.cu): one new position per sequence.
// p_dev (optional): read the position from the device instead of p (CUDA-graph decode steps)
void embed_rows(const int32_t* ids, const float* tok, const float* pos, int p, float* x, int B, int d, cudaStream_t s,
                const int* p_dev = nullptr);
void kv_scatter(const bf16* qkv_new, bf16* cache, int B, int T, int p, int dl, cudaStream_t s,
                const int* p_dev = nullptr);
void bump_i32(int* x, cudaStream_t s);  // *x += 1 on the device
void decode_attention(const bf16* qkv_new, const bf16* cache, bf16* out, int B, int T, int p, int Hl, int hd,
                      cudaStream_t s, const int* p_dev = nullptr);
// Split-key decode attention for head_dim 64 / 128 / 256 with the kv_scatter of the new row
// fused in (returns false for other head dims): part holds B*Hl*decode_split_count()*(hd+2)
// floats, ticket B*Hl zero-initialised counters (never reset)
bool decode_attention_split(const bf16* qkv_new, bf16* cache, bf16* out, int B, int T, int p, int Hl, int hd,
                            cudaStream_t s, const int* p_dev, float* part, unsigned int* ticket);
int decode_split_count();
// scratch (optional, B * kArgmaxChunks * 2 floats): split each row over up to kArgmaxChunks CTAs
constexpr int kArgmaxChunks = 64;
void argmax_rows(const bf16* x, int64_t row_stride, int B, int n, int index_base, float* out, cudaStream_t s,
                 float* scratch = nullptr);
void argmax_combine(const float* parts, int shards, int B, int32_t* tok, cudaStream_t s);

void sum_f32(const float* x, int64_t n, float* out, cudaStream_t s);
// Fused softmax cross entropy forward + backward over the vocab (kernels.hpp:327-363):
// wloss[m] = w[m] * (logsumexp - logit[target]); logits <- (softmax - onehot) * w[m] / wsum.
void xent_fwd_bwd(bf16* logits, int64_t ld, int64_t M, int V, const int32_t* targets,
                  const float* weights, const float* wsum, float* wloss, int write_grad,
                  cudaStream_t s);
// Vocab-parallel cross entropy (logits split along the vocab across mp ranks; the lm_head
// split:0 override of SURVEY D1). Rank-local pass: stats[2m] = local max, stats[2m+1] = sum of
// exp(x - max); tlogit[m] = logit of the target if this rank owns it, else 0.
void xent_vp_stats(const bf16* logits, int64_t ld, int64_t M, int Vl, int v0, const int32_t* targets,
                   float* stats, float* tlogit, cudaStream_t s);
// After gathering every rank's stats ([t][M*2]) and summing tlogit: lse[m], wloss[m].
void xent_vp_combine(const float* stats_all, int t, int64_t M, const float* tlogit, const float* weights,
                     float* lse, float* wloss, cudaStream_t s);
// logits <- (exp(x - lse) - onehot) * w / wsum on the local vocab slice.
void xent_vp_grad(bf16* logits, int64_t ld, int64_t M, int Vl, int v0, const int32_t* targets, const float* lse,
                  const float* weights, const float* wsum, cudaStream_t s);
// loss[0] = sum(wloss) / wsum (double)
// loss = sum(wloss) / wsum; a non-finite loss ORs 2 into *gate (when given): the fused
// optimizer epilogues of the following backward then leave the state untouched
void loss_reduce(const float* wloss, int64_t M, const float* wsum, double* loss, cudaStream_t s,
                 int* gate = nullptr);

// Causal scaled-dot-product attention on the head-sharded QKV activations:
// qkv [M, 3*Dl] (q | k | v, head h at column h*hd), o [M, Dl], lse [B, Hl, T]
// (graph.hpp:650-661 with the -1e9 causal mask of model.hpp:100-106).
void attention_trace_read(unsigned long long* out);
void attention_fwd(const bf16* qkv, bf16* o, float* lse, int B, int T, int Hl, int hd,
                   cudaStream_t s);
// dqkv [M, 3*Dl]; scratch: attention_bwd_scratch_floats(B, T, Hl, hd) fp32 elements (delta, and
// the fp32 dQ accumulator or, for head_dim 128 with T % 128 == 0, the dS^T tiles of the dQ kernel).
// delta_ready: scratch already holds delta = rowsum(dO * O) (written by the dO GEMM's kBf16Delta
// epilogue), so the tcgen05 path skips its delta pass.
// colsum (optional, [M / 32][3*Dl] fp32): the q|k|v bias gradients' per-32-row column partials
// of dqkv, written when *colsum_done comes back true (reduce with colsum_chunks).
int64_t attention_bwd_scratch_floats(int B, int T, int Hl, int hd);
void attention_bwd(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, bf16* dqkv,
                   float* scratch, int B, int T, int Hl, int hd, cudaStream_t s, bool delta_ready = false,
                   float* colsum = nullptr, bool* colsum_done = nullptr);

// y = a + b + bias[col]   (row-parallel output after the all-reduce: residual + partial + bias)
void add_residual_bias(const float* a, const float* b, const float* bias, float* y, int64_t M,
                       int d, cudaStream_t s);
void add_residual_bias(const float* a, const bf16* b, const float* bias, float* y, int64_t M, int d,
                       cudaStream_t s);

// AdamW over a flat shard (train_state.hpp:183-220, Scalar = float); also refreshes the bf16
// shadow copy used by the GEMMs.
// gate (optional): skip the update when *gate != 0 (read on the device)
void adamw(float* p, float* m, float* v, const float* g, bf16* shadow, int64_t n, float lr,
           float b1, float b2, float eps, float wd, float c1, float c2, cudaStream_t s,
           const int* gate = nullptr);
// flag[0] |= any non-finite among x[0..n)
void nonfinite_check(const float* x, int64_t n, int* flag, cudaStream_t s);
void scale_f32(float* x, int64_t n, float a, cudaStream_t s);
void cast_f32_bf16(const float* x, bf16* y, int64_t n, cudaStream_t s);
void cast_bf16_f32(const bf16* x, float* y, int64_t n, cudaStream_t s);

// ---- T5 encoder-decoder extension (t5_kernels.cu) ----
// q / k / v / o: bf16 rows of B*T tokens (row pitch ld*), head h at column h*dk; lse [B, Hl, Tq];
// bias [Hl, Tq, Tk] fp32 or null; scores = scale * q.k (+ bias) (+ causal mask).
struct T5AttnArgs {
  const bf16* q = nullptr;
  int64_t ldq = 0;
  const bf16* k = nullptr;
  int64_t ldk = 0;
  const bf16* v = nullptr;
  int64_t ldv = 0;
  bf16* o = nullptr;
  int64_t ldo = 0;
  float* lse = nullptr;
  const float* bias = nullptr;
  int Tq = 0, Tk = 0, Hl = 0, dk = 0, causal = 0;
  float scale = 1.f;
};
void t5_attention_fwd(const T5AttnArgs& a, int B, cudaStream_t s);
// dq (bf16, pitch lddq) written; dk / dv (bf16) written from fp32 atomics; dbias (fp32
// [Hl, Tq, Tk], may be null) accumulated. scratch: t5_attention_scratch floats.
void t5_attention_bwd(const T5AttnArgs& a, int B, const bf16* dout, int64_t ldd, bf16* dq, int64_t lddq, bf16* dk,
                      int64_t lddk, bf16* dv, int64_t lddv, float* scratch, float* dbias, cudaStream_t s);
int64_t t5_attention_scratch(int B, int Hl, int Tq, int Tk, int dk);
// bias[h, i, j] = table[ids[i, j], h0 + h] for the rank's Hl heads (table [buckets, H])
void t5_bias_build(const float* table, const int32_t* ids, int H, int h0, int Hl, int64_t TT, float* bias,
                   cudaStream_t s);
// table_grad[bucket, h0 + h] += sum over positions with that bucket of dbias[h]
void t5_bias_grad(const float* dbias, const int32_t* ids, int H, int h0, int Hl, int64_t TT, int nb,
                  float* table_grad, cudaStream_t s);
// tcgen05 attention over fused q|k|v activations in the general form the T5 extension needs:
// causal or not, optional relative-position bias lut [Hl][2T + 128] (index key - query + T - 1,
// natural units), score scale; the backward adds the bias gradient into dlut. Returns false
// (nothing launched) when the shape is not covered (head dim != 128, T + 128 > 4096 with a lut).
bool attention_fwd_ex(const bf16* qkv, bf16* o, float* lse, int B, int T, int Hl, int hd, int causal,
                      const float* lut, float scale, cudaStream_t s);
bool attention_bwd_ex(const bf16* qkv, const bf16* o, const float* lse, const bf16* dout, bf16* dqkv,
                      float* scratch, int B, int T, int Hl, int hd, int causal, const float* lut, float* dlut,
                      float scale, cudaStream_t s);
// Cross-attention on the tensor cores (head_dim 128, non-causal, no bias): q [B*Tq] rows of
// pitch ldq, k | v [B*Tk] rows of pitch ldkv with v at +voff; backward writes dq (pitch ld_dq)
// and dk | dv (pitch ld_dkv, dv at +voff). false = not handled (use the CUDA-core kernels).
bool attention_fwd_cross(const bf16* q, int64_t ldq, const bf16* kv, int64_t ldkv, int voff, bf16* o, float* lse,
                         int B, int Tq, int Tk, int Hl, int hd, float scale, cudaStream_t s);
bool attention_bwd_cross(const bf16* q, int64_t ldq, const bf16* kv, int64_t ldkv, int voff, const bf16* o,
                         const float* lse, const bf16* dout, bf16* dq, int64_t ld_dq, bf16* dkv, int64_t ld_dkv,
                         float* scratch, int B, int Tq, int Tk, int Hl, int hd, float scale, cudaStream_t s);
// lut[h][d + T - 1] = table[bucket[d + T - 1], h0 + h] for d in (-T, T); zero padding to 2T + 128
void t5_lut_build(const float* table, const int32_t* bucket, int H, int h0, int Hl, int T, float* lut, cudaStream_t s);
// table_grad[bucket[i], h0 + h] += dlut[h][i] for i < 2T - 1
void t5_lut_grad(const float* dlut, const int32_t* bucket, int H, int h0, int Hl, int T, float* table_grad,
                 cudaStream_t s);

// Emulated collective: every bufs[r][0..n) <- sum_{r ascending} bufs[r] (collectives.hpp:27-52).
void sum_ranks_f32(float* const* bufs, int nranks, int64_t n, float scale, cudaStream_t s);
void sum_ranks_bf16(bf16* const* bufs, int nranks, int64_t n, float scale, cudaStream_t s);

// init_transformer_params on the device (model.hpp:49-70 + rng.hpp:15-91): element (r, c) of
// the FULL [rows, cols] tensor takes normal draw number base_draw/2 + r*cols + c of the stream
// with key `key`, times `scale`. The local shard covers rows [r0, r0+lr) x cols [c0, c0+lc).
void init_normal(float* out, int64_t lr, int64_t lc, int64_t r0, int64_t c0, int64_t cols,
                 uint64_t key, uint64_t base_counter, double scale, cudaStream_t s);
void fill_f32(float* out, int64_t n, float v, cudaStream_t s);

}  // namespace k
}  // namespace sw
