// GPU executor of the T5 encoder-decoder extension (BASELINE cfg4).
//
// The reference has no encoder-decoder model; this executes the T5 v1.0 step composed from the
// reference's ops (oracle/t5_ref.py states it) under the plan the reference's rules derive for
// the T5 parameter tree (rules.h t5 keys): q/k/v of self- and cross-attention column-split,
// o row-split, fc1 column-split, fc2 row-split; rel_bias, embeddings, norms and lm_head
// replicated. Per device the state is the same five flat buffers as Model (fp32 p/g/m/v + bf16
// shadow); q|k|v of a self-attention block are adjacent (one fused QKV GEMM) and k|v of a
// cross-attention block are adjacent (one fused KV GEMM over the encoder output).
//
// Scope: dp = 1 (tensor parallel over the mesh's mp axis, emulated or NCCL), replicated lm_head.
// The GEMMs are the tcgen05 family (the MLP's ReLU and its derivative in their epilogues);
// train_step applies AdamW inside the weight-gradient GEMM epilogues (GEMM weights, region 1 of
// the flat layout) and one flat AdamW over the rest. Attention: the tcgen05 kernels of
// attention_mma.cu for d_kv = 128 (relative bias as a per-head LUT, cross-attention over the
// encoder K/V), the CUDA-core kernels of t5_kernels.cu otherwise.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <string>
#include <unordered_map>
#include <vector>

#include "mesh.h"
#include "model.h"
#include "rules.h"

namespace sw {

struct T5Layer {
  int ln1 = -1, q = -1, o = -1, lnx = -1, cq = -1, ck = -1, co = -1, ln2 = -1, fc1 = -1, fc2 = -1;
};

struct T5Rank {
  int device = 0, mpi = 0;
  float *p = nullptr, *g = nullptr, *m = nullptr, *v = nullptr;
  bf16* w = nullptr;
  // encoder activations (per layer) and output
  std::vector<float*> hs_e, hm_e, st1_e, st2_e;
  std::vector<bf16*> a1_e, qkv_e, o_e, a2_e, act_e;
  std::vector<float*> lse_e;
  float* stf_e = nullptr;
  bf16* eo = nullptr;
  // decoder activations
  std::vector<float*> hs_d, hm_d, hx_d, st1_d, stx_d, st2_d;
  std::vector<bf16*> a1_d, qkv_d, o_d, ax_d, cq_d, ckv_d, co_d, a2_d, act_d;
  std::vector<float*> lse_d, clse_d;
  float* stf_d = nullptr;
  bf16 *f = nullptr, *logits = nullptr;
  // relative-position bias (this rank's heads) and its gradient
  int32_t *ids_e = nullptr, *ids_d = nullptr;
  float *bias_e = nullptr, *bias_d = nullptr, *dbias_e = nullptr, *dbias_d = nullptr;
  // tcgen05 path: the bias as a per-head LUT over key - query ([Hl][2T + 128]) and its gradient
  int32_t *bd_e = nullptr, *bd_d = nullptr;  // bucket of each offset key - query + T - 1
  float *lut_e = nullptr, *lut_d = nullptr, *dlut_e = nullptr, *dlut_d = nullptr;
  // inputs
  int32_t *enc_tok = nullptr, *dec_tok = nullptr, *targets = nullptr;
  float *weights = nullptr, *wloss = nullptr, *wsum = nullptr;
  double* loss = nullptr;
  // backward scratch
  float *gres_e = nullptr, *gres_d = nullptr, *dx = nullptr, *part = nullptr, *d_eout = nullptr;
  bf16 *gb = nullptr, *dqkv = nullptr, *dout = nullptr, *dact = nullptr, *dcq = nullptr, *dckv = nullptr;
  float *attn_scratch = nullptr, *ln_partials = nullptr;
  uint32_t* tok_keys = nullptr;
};

class T5Model {
 public:
  T5Model(const ModelSpec& spec, const Plan& plan, Mesh* mesh, int batch, int enc_len, int dec_len);
  ~T5Model();

  void init_params(uint64_t seed, const std::string& stream_name);
  void set_tensor(const std::string& name, int which, const float* full, int64_t numel);
  void get_tensor(const std::string& name, int which, float* full, int64_t numel);
  // enc [batch, enc_len], dec / targets / weights [batch, dec_len] (weights may be null = 1)
  void stage_batch(const int32_t* enc, const int32_t* dec, const int32_t* targets, const float* weights);
  void forward_backward();
  void forward_only();
  void adamw(double lr, double b1, double b2, double eps, double wd);
  // forward_backward + adamw with the optimizer fused into the weight-gradient GEMMs (dp = 1,
  // as Model::train_step; SW_FUSED_ADAMW=0: the two-pass step). Returns whether it was fused.
  bool train_step(double lr, double b1, double b2, double eps, double wd);
  double last_loss();
  void logits_to_host(float* out);  // [batch * dec_len, vocab] of mp rank 0
  uint64_t step() const { return step_; }

  cudaStream_t stream() const { return stream_; }
  int64_t launches() const { return launches_; }
  int64_t device_bytes() const { return bytes_; }
  void set_profiling(bool on);
  void read_profile(double* ms, double* work, int64_t* count);

 private:
  template <typename T>
  T* alloc(int64_t n);
  void build_layout();
  void allocate();
  void forward(bool need_grad);
  void backward();
  // relu: the MLP's ReLU in the epilogue (kStoreBf16 / kGeluBwd with GemmParams::relu)
  void gemm(int M, int N, int K, const void* A, int64_t lda, int a_mn, const void* B, int64_t ldb, int b_mn,
            int epi, void* C, int64_t ldc, const void* aux = nullptr, int64_t ld_aux = 0, int accumulate = 0,
            int relu = 0);
  // weight gradient dW[M, N] = A^T B (MN-major operands) into G, or with fused_ set the AdamW
  // update of the slot in the GEMM epilogue
  void wgrad(T5Rank& R, int slot, int M, int N, int K, const void* A, int64_t lda, const void* B, int64_t ldb);
  struct FusedAdam {
    float lr, b1, b2, eps, wd, c1, c2;
  };
  const FusedAdam* fused_ = nullptr;
  int* d_flag_ = nullptr;
  int64_t weights_end_ = 0;  // [0, weights_end_): GEMM weight matrices
  bool poisoned_ = false;  // a fused step updated some weights before finding a non-finite gradient
  void check_not_poisoned(const char* what) const;
  // all-reduce (sum) over the mp group of n floats at ptr(R) of every local rank
  void ar(const std::function<float*(T5Rank&)>& ptr, int64_t n);
  // row-parallel product [M, K] x W[d, K]^T added to the residual `aux` into `out`
  void row_parallel(int64_t M, int K, const std::function<const bf16*(T5Rank&)>& a, int w_slot,
                    const std::function<const float*(T5Rank&)>& aux, const std::function<float*(T5Rank&)>& out);
  void attn_fwd(T5Rank& R, int Tq, int Tk, const bf16* q, int64_t ldq, const bf16* k, const bf16* v,
                int64_t ldkv, bf16* o, float* lse, const float* bias, int causal);
  void rms_fwd(const float* x, int scale_slot, T5Rank& R, bf16* y, float* rstd, int64_t M);
  void rms_bwd(const float* x, const float* rstd, int scale_slot, T5Rank& R, const float* dy, float* gres,
               int64_t M, int accumulate);
  float* P(T5Rank& R, int s) { return R.p + slots_[s].offset; }
  float* G(T5Rank& R, int s) { return R.g + slots_[s].offset; }
  bf16* W(T5Rank& R, int s) { return R.w + slots_[s].offset; }
  void tic();
  void toc(int cat, double work);

  ModelSpec spec_;
  Plan plan_;
  Mesh* mesh_;
  int B_, Te_, Td_;
  int64_t Me_, Md_;
  int Le_, Ld_, d_, H_, dk_, inner_, dff_, V_, nb_, maxd_;
  int t_ = 1, hl_ = 0, il_ = 0, fl_ = 0;
  // Te == Td: cross-attention q | k | v share one [B*T, 3*inner/t] buffer (the q GEMM writes
  // columns [0, inner/t), the k|v GEMM over the encoder output the rest), which is the fused
  // layout the tcgen05 attention reads; tc_: head dim 128 and Te == Td (SW_T5_TC=0 forces the
  // CUDA-core kernels)
  bool fused_x_ = false, tc_ = false;
  int64_t ld_cq_ = 0, ld_ckv_ = 0;
  std::vector<Slot> slots_;
  std::unordered_map<std::string, int> slot_of_;
  std::vector<T5Layer> enc_, dec_;
  int tok_ = -1, rb_e_ = -1, rb_d_ = -1, lnf_e_ = -1, lnf_d_ = -1, head_ = -1;
  int64_t flat_n_ = 0;
  std::vector<T5Rank> ranks_;
  std::vector<void*> allocations_;
  cudaStream_t stream_ = nullptr;
  int64_t launches_ = 0;
  int64_t bytes_ = 0;
  uint64_t step_ = 0;
  bool prof_ = false;
  std::vector<cudaEvent_t> events_;
  size_t ev_next_ = 0;
  std::vector<std::pair<int, double>> prof_rec_;
};

}  // namespace sw
