// GPU executor of the tensor-parallel transformer step.
//
// Replaces, for the transformer_loss program (model.hpp:144-152), the reference's
// SpmdInterpreter::run / spmd_forward_backward (spmd.hpp:96-119, :782-814), the shard
// materialiser shard_params / replica_param_views / gather_params (train_state.hpp:50-110),
// dp_sync_grads (:155-170) and adamw_step (:183-220).
//
// Per device ("rank") the state is five flat buffers over that rank's parameter shards
// (fp32 master params, grads, Adam m, Adam v; bf16 shadow for the GEMMs), laid out so that
// every GEMM operand is one contiguous, TMA-addressable matrix: the q, k, v kernel shards of a
// layer are adjacent ([3*d/t, d] fused QKV) and their replicated biases are adjacent ([3*d]).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <string>
#include <unordered_map>
#include <vector>

#include "checkpoint.h"
#include "mesh.h"
#include "rules.h"

namespace sw {

using bf16 = __nv_bfloat16;

struct Slot {
  std::string name;
  Dims global, local;
  Layout layout;
  int64_t begin = 0, end = 0;  // owned range along the split dim
  int64_t offset = 0;          // element offset in the rank's flat buffers
  int64_t numel = 0;           // local elements
  int init = 0;                // 0 zeros, 1 ones, 2 normal
  double init_scale = 0.0;
  uint64_t draw_base = 0;      // counter of the slot's first draw in the init stream
};

// Slot indices of one block; -1 = absent (RMSNorm has no bias, the SwiGLU MLP has no biases).
// With SwiGLU, gate_k and fc1_k (up) are adjacent: the fused [gate; up] weight starts at gate_k.
struct LayerSlots {
  int ln1_s = -1, ln1_b = -1, q_k = -1, k_k = -1, v_k = -1, q_b = -1, k_b = -1, v_b = -1, o_k = -1, o_b = -1,
      ln2_s = -1, ln2_b = -1, gate_k = -1, fc1_k = -1, fc1_b = -1, fc2_k = -1, fc2_b = -1;
};

struct Rank {
  int device = 0, dpi = 0, mpi = 0;
  // inference-only model: p, g, m, v null; p_small holds the region-2 parameters (flat offsets
  // >= weights_end_), the GEMM weights live in w only
  float *p = nullptr, *g = nullptr, *m = nullptr, *v = nullptr;
  float* p_small = nullptr;
  bf16* w = nullptr;
  // activations saved for the backward, per layer
  std::vector<float*> hs, hmid, stats1, stats2;  // stats: mean[M] | rstd[M]
  std::vector<bf16*> a1, a2, qkv, o, pre, act;
  std::vector<float*> lse;
  float* statsf = nullptr;
  bf16* f = nullptr;
  bf16* logits = nullptr;
  // inputs
  int32_t *tokens = nullptr, *targets = nullptr;
  float* weights = nullptr;
  float *wloss = nullptr, *wsum = nullptr;
  double* loss = nullptr;
  // scratch
  float *part = nullptr, *dx = nullptr, *gres = nullptr, *col_scratch = nullptr, *attn_scratch = nullptr;
  float* ln_partials = nullptr;  // per-CTA LayerNorm parameter-gradient partials (deterministic reduction)
  uint32_t* tok_keys = nullptr;  // sorted (token, position) keys of the embedding backward
  // vocab-parallel cross entropy: per-rank (max, sumexp) of every mp rank, target logit, lse
  float *xstats = nullptr, *xt = nullptr, *xlse = nullptr;
  bf16 *gb = nullptr, *dpre = nullptr, *dout = nullptr, *dqkv = nullptr;
  bf16* arb = nullptr;  // [M, d] bf16 payload of the row-parallel all-reduces (ar_bf16)
};

// Kernel categories of the per-launch profile (CUDA events around each launch, read back
// after a synchronize). `work` is algorithmic FLOPs for GEMM/attention and algorithmic HBM
// bytes for the memory-bound kernels.
enum ProfCat : int {
  kProfGemm = 0,
  kProfAttnFwd = 1,
  kProfAttnBwd = 2,
  kProfNorm = 3,
  kProfXent = 4,
  kProfAdamw = 5,
  kProfComm = 6,
  kProfOther = 7,
  kProfCats = 8
};

class Model {
 public:
  // inference = true: an inference-only model (generate / forward_only / logits; see allocate):
  // bf16 GEMM weights + fp32 small parameters + the K/V cache, about a ninth of the training
  // footprint, so an OPT-66B-shape model fits one B200 (cfg5).
  Model(const ModelSpec& spec, const Plan& plan, Mesh* mesh, int batch, int seq_len, bool inference = false);
  ~Model();

  void init_params(uint64_t seed, const std::string& stream_name);
  void set_param(const std::string& name, const float* full, int64_t numel);
  // which: 0 param (+ bf16 shadow), 2 adam_m, 3 adam_v
  void set_tensor(const std::string& name, int which, const float* full, int64_t numel);
  // SWCK snapshots (checkpoint.hpp:193-298): replica 0's gathered p / m / v in tree order;
  // load re-cuts them onto this model's plan and mesh.
  void save_checkpoint(const std::string& path, const std::vector<CkptRng>& rngs);
  void load_checkpoint(const std::string& path);
  const std::vector<CkptRng>& loaded_rngs() const { return loaded_rngs_; }
  // Greedy next-token generation (the Predictor loop of cli.cpp:425-447): prompts [batch, P]
  // (every row P tokens), n_new tokens per row into out [batch, n_new]. While the context fits
  // the seq_len window the step runs one position through a KV cache (the layer's qkv
  // activations); once it slides, the window is re-run with positions 0..T-1 exactly as the
  // reference does.
  void generate(const int32_t* prompts, int P, int n_new, int32_t* out);
  uint64_t step() const { return step_; }
  uint64_t seed() const { return seed_; }
  void get_tensor(const std::string& name, int which, float* full, int64_t numel);
  void stage_batch(const int32_t* tokens, const int32_t* targets, const float* weights);
  void forward_backward(bool accumulate);
  void forward_only();
  void scale_grads(double factor);
  void dp_sync();
  void adamw(double lr, double b1, double b2, double eps, double wd, bool check_finite);
  // forward_backward + dp_sync + adamw; with dp == 1 the optimizer runs inside the backward
  // (wgrad epilogues). Returns true when the fused path ran.
  // A non-finite loss gates every fused update (the step is then redone unfused, so the state is
  // unchanged when NonFiniteError names the parameter, as train_state.hpp:207-210 does). A
  // non-finite gradient under a finite loss is found only inside the backward, after some
  // epilogues updated their weights: the model is then poisoned (train_step, forward_backward,
  // adamw and save_checkpoint refuse) until init_params or load_checkpoint.
  bool train_step(double lr, double b1, double b2, double eps, double wd);
  bool poisoned() const { return poisoned_; }
  bool inference() const { return inference_; }
  double last_loss();
  void logits_to_host(float* out);

  cudaStream_t stream() const { return stream_; }
  int64_t launches() const { return launches_; }
  void reset_launches() { launches_ = 0; }
  void set_profiling(bool on);
  // Per category: summed device milliseconds, summed work, launch count (since the last read).
  void read_profile(double* ms, double* work, int64_t* count);
  int64_t device_bytes() const { return bytes_; }

 private:
  void check_not_poisoned(const char* what) const;
  void check_trainable(const char* what) const;  // refuses on an inference-only model
  template <typename T>
  T* alloc(int64_t n);
  void build_layout();
  void allocate();
  std::vector<Rank*> replica(int dpi);
  void forward_replica(std::vector<Rank*>& grp, bool need_grad);
  void backward_replica(std::vector<Rank*>& grp, bool accumulate);
  void ar_mp(std::vector<Rank*>& grp, float* Rank::*buf, int64_t n);
  void ar_mp_ptrs(std::vector<Rank*>& grp, const std::vector<float*>& ptrs, int64_t n, cudaStream_t s = nullptr);
  // Row-parallel product + all-reduce + consumer, pipelined over row chunks: the producer of
  // chunk c+1 runs on the compute stream while chunk c is all-reduced on the comm stream.
  using RowFn = std::function<void(Rank&, int64_t r0, int64_t rows)>;
  void row_parallel_ar(std::vector<Rank*>& grp, float* Rank::*buf, int width, const RowFn& produce,
                       const RowFn& consume);
  void row_parallel_ar(std::vector<Rank*>& grp, bf16* Rank::*buf, int width, const RowFn& produce,
                       const RowFn& consume);
  void ar_mp_ptrs(std::vector<Rank*>& grp, const std::vector<bf16*>& ptrs, int64_t n, cudaStream_t s);
  // Row-parallel GEMM (A [rows, K] x W^T) + all-reduce of the [M, d] output + consumer, with the
  // payload in fp32 (`f32buf`) or, when ar_bf16_, in bf16 (Rank::arb). The consumer receives the
  // reduced rows as either type.
  using ConsFn = std::function<void(Rank&, int64_t r0, int64_t rows, const float* f32, const bf16* b16)>;
  void row_ar(std::vector<Rank*>& grp, float* Rank::*f32buf, const std::function<const bf16*(Rank&)>& a,
              int64_t lda, int K, int w_slot, int b_mn, const ConsFn& consume);
  void ag_mp_slot(std::vector<Rank*>& grp, int slot, int64_t chunk);
  // in-place all-gather: chunk `mpi` of base(R) is local, the others arrive from the peers
  void ag_mp_buf(std::vector<Rank*>& grp, float* Rank::*buf, int64_t chunk);
  void gemm(Rank& R, int M, int N, int K, const void* A, int64_t lda, int a_mn, const void* B,
            int64_t ldb, int b_mn, int epi, void* C, int64_t ldc, void* C2 = nullptr,
            int64_t ldc2 = 0, const float* bias = nullptr, const void* aux = nullptr,
            int64_t ld_aux = 0, int accumulate = 0, int bias_seg = 0, int64_t bias_seg_stride = 0,
            int swiglu_half = 0, float* delta = nullptr, int delta_T = 0, float* colsum = nullptr);
  // dO = gb x Wo with the attention backward's delta = rowsum(dO * O) fused into the epilogue
  // (kBf16Delta) when the GEMM path supports it; returns whether delta was written
  bool gemm_dout(Rank& R, int l, const bf16* wo);
  void wgrad(Rank& R, int slot, int M, int N, int K, const void* A, int64_t lda, const void* B, int64_t ldb,
             int accumulate);
  struct FusedAdam {
    float lr, b1, b2, eps, wd, c1, c2;
  };
  const FusedAdam* fused_ = nullptr;
  // fp32 parameter at a flat offset (an inference-only model keeps region 2 only)
  float* pval(Rank& R, int64_t offset) {
    if (R.p != nullptr) return R.p + offset;
    if (offset < weights_end_) fail_no_fp32_weight();
    return R.p_small + (offset - weights_end_);
  }
  [[noreturn]] static void fail_no_fp32_weight();
  float* P(Rank& R, int slot) { return pval(R, slots_[slot].offset); }
  float* Pn(Rank& R, int slot) { return slot < 0 ? nullptr : P(R, slot); }  // absent slot -> null
  float* Gn(Rank& R, int slot) { return slot < 0 ? nullptr : G(R, slot); }
  float* G(Rank& R, int slot) { return R.g + slots_[slot].offset; }
  bf16* W(Rank& R, int slot) { return R.w + slots_[slot].offset; }

  ModelSpec spec_;
  Plan plan_;
  Mesh* mesh_;
  int B_, T_;
  int64_t M_;
  int L_, d_, H_, hd_, dff_, V_, S_;
  int ta_ = 1, tm_ = 1, th_ = 1;  // TP degree of attention, MLP, LM head (1 = replicated)
  int dl_, hl_, fl_, vl_, ldv_;
  std::vector<Slot> slots_;
  std::unordered_map<std::string, int> slot_of_;
  std::vector<LayerSlots> layers_;
  int tok_ = -1, pos_ = -1, lnf_s_ = -1, lnf_b_ = -1, head_ = -1;
  int64_t flat_n_ = 0;
  int64_t weights_end_ = 0;  // [0, weights_end_): GEMM weight matrices; the rest: small params
  std::vector<Rank> ranks_;
  std::vector<void*> allocations_;
  cudaStream_t stream_ = nullptr;
  cudaStream_t comm_stream_ = nullptr;
  // Weight-gradient GEMMs run on side_ (SW_WGRAD_STREAM=0: on stream_), forked after their
  // inputs are written and joined before those inputs are overwritten, so a wgrad's last
  // partial wave of tiles shares the SMs with the next dgrad / attention kernel.
  cudaStream_t side_ = nullptr;
  std::vector<cudaEvent_t> side_ev_;  // grows on demand; reused from index 0 every backward
  size_t side_next_ = 0;
  cudaEvent_t on_side(const std::function<void()>& f);
  void main_wait(cudaEvent_t e);
  // dp gradient all-reduce overlapped with the backward (train_step with dp > 1): layer l's
  // GEMM-weight gradients (a contiguous range of region 1) are all-reduced on dp_stream_ as soon
  // as its last weight-gradient GEMM is done; dp_sync then reduces only the rest
  bool dp_overlap_ = false;
  bool dp_buckets_issued_ = false;
  cudaStream_t dp_stream_ = nullptr;
  std::vector<cudaEvent_t> dp_ev_;
  int64_t layers_end_ = 0;  // end of the last layer's GEMM weights in the flat layout
  void dp_reduce_range(int64_t off, int64_t n, cudaStream_t s);
  void dp_bucket(std::vector<Rank*>& grp, int l, cudaEvent_t ready);
  std::vector<cudaEvent_t> ev_prod_, ev_ar_;
  int ar_chunks_ = 1;
  // Row-parallel all-reduce payloads in bf16 (opt-in, SW_AR_BF16=1): half the NVLink bytes of
  // the fp32 partials, but the partials and the sum are rounded to bf16. Off by default: the
  // oracle-parity tolerances of the mini configurations (LayerNorm parameter gradients at 1e-2)
  // do not survive it; TP invariance on tiny.spec does (tests/test_model_gpu.py).
  bool ar_bf16_ = false;
  bool fuse_colsum_ = true;  // SW_FUSE_COLSUM=0: fc1 bias gradient by the separate column-sum pass
  int* d_flag_ = nullptr;
  int64_t launches_ = 0;
  // profiling
  void tic(cudaStream_t s = nullptr);
  void toc(int cat, double work, cudaStream_t s = nullptr);
  bool prof_ = false;
  std::vector<cudaEvent_t> events_;
  size_t ev_next_ = 0;
  std::vector<std::pair<int, double>> prof_rec_;
  std::vector<std::string> prof_tag_;  // per record: GEMM shape / epilogue (SW_PROFILE_LOG dump)
  int64_t bytes_ = 0;
  uint64_t step_ = 0;
  bool poisoned_ = false;
  bool inference_ = false;
  uint64_t seed_ = 0;
  struct DecodeBufs {
    float *x = nullptr, *xmid = nullptr, *part = nullptr, *stats = nullptr, *arg = nullptr;
    bf16 *a = nullptr, *qkv = nullptr, *o = nullptr, *pre = nullptr, *h = nullptr, *f = nullptr, *logits = nullptr;
    int32_t* tok = nullptr;
    int* pos = nullptr;  // device position of the cached step (read by the CUDA-graph step)
    float* attn_part = nullptr;       // split-key decode attention partials
    unsigned int* attn_ticket = nullptr;
    float* argpart = nullptr;  // per-chunk argmax winners
  };
  std::vector<DecodeBufs> dec_;  // per local rank, allocated on the first generate()
  int32_t* dec_out_ = nullptr;   // [n_cap, B] tokens of cached steps, read back in batches
  int64_t dec_out_cap_ = 0;
  cudaGraphExec_t dec_graph_ = nullptr;  // one cached decode step, position on the device
  // prefill (window_forward): >= 0 makes forward_replica compute the logits of only this row of
  // every sequence, into the decode buffers, and skip the loss
  int head_row_ = -1;
  int head_seq_ = 0;  // the decode-buffer row its logits go to (one-sequence-at-a-time prefill)
  // decode_step: small-M GEMMs launched as programmatic dependents (0 off; 1 + n: n x U weight
  // steps requested into L2 before griddepcontrol.wait)
  int pdl_ = 0;
  // p >= 0: position p (host value); p < 0: every rank's dec_[].pos, advanced at the step's end
  void decode_step(std::vector<Rank*>& grp, int p);
  void window_forward(std::vector<Rank*>& grp, const std::vector<std::vector<int32_t>>& ctx, int take);
  // moves every per-token activation pointer of the group by `rows` token rows (the prefill runs
  // one sequence at a time over the first rows of its window, see window_forward)
  void shift_rows(std::vector<Rank*>& grp, int64_t rows);
  // argmax of one logits row per sequence (per-rank base pointer, row stride in elements) into
  // every rank's dec_[].tok, combining vocab shards when the head is split
  void pick_tokens(std::vector<Rank*>& grp, const std::vector<const bf16*>& rows, int64_t stride);
  std::vector<CkptRng> loaded_rngs_;
};

}  // namespace sw
