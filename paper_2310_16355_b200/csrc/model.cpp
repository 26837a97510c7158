// GPU executor of the tensor-parallel transformer step (see model.h).
#include "model.h"

#include <unordered_map>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "gemm.h"
#include "kernels.h"
#include "status.h"

namespace sw {

namespace {

uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 0x100000001b3ull;
  }
  return h;
}

int64_t numel_of(const Dims& d) {
  int64_t n = 1;
  for (int64_t x : d) n *= x;
  return n;
}

constexpr int64_t kAlign = 64;  // elements; keeps every slot 256-B aligned in fp32, 128-B in bf16

}  // namespace

// ---------------------------------------------------------------------------------------------
// construction: plan -> per-rank layout
// ---------------------------------------------------------------------------------------------
Model::Model(const ModelSpec& spec, const Plan& plan, Mesh* mesh, int batch, int seq_len, bool inference)
    : spec_(spec), plan_(plan), mesh_(mesh), B_(batch), T_(seq_len), inference_(inference) {
  if (mesh == nullptr) fail(SW_ERR_CONFIG, "sw_model_create: mesh is NULL");
  if (batch < 1 || seq_len < 1) {
    fail(SW_ERR_CONFIG, "transformer_logits: batch and seq_len must be positive");
  }
  if (seq_len > spec.max_seq_len) {
    fail(SW_ERR_CONFIG, "transformer_logits: seq_len " + std::to_string(seq_len) +
                            " exceeds max_seq_len " + std::to_string(spec.max_seq_len));
  }
  if (plan.n_shards != mesh->mp) {
    fail(SW_ERR_CONFIG, "sw_model_create: plan has n_shards=" + std::to_string(plan.n_shards) +
                            " but the mesh has mp=" + std::to_string(mesh->mp));
  }
  M_ = static_cast<int64_t>(B_) * T_;
  L_ = spec.n_layers;
  d_ = static_cast<int>(spec.d_model);
  H_ = spec.n_heads;
  hd_ = d_ / H_;
  dff_ = static_cast<int>(spec.d_ff);
  V_ = static_cast<int>(spec.vocab_size);
  S_ = static_cast<int>(spec.max_seq_len);
  cuda_check(cudaSetDevice(mesh->cuda_device), "cudaSetDevice");
  cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  cuda_check(cudaStreamCreateWithFlags(&comm_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  {
    const char* e = std::getenv("SW_AR_BF16");
    ar_bf16_ = mesh_->mp > 1 && e != nullptr && e[0] == '1';
    const char* fc = std::getenv("SW_FUSE_COLSUM");
    fuse_colsum_ = fc == nullptr || fc[0] != '0';
  }
  build_layout();
  allocate();
  // all-reduce pipelining depth (SW_AR_CHUNKS overrides): 4 row chunks when they stay 128-aligned
  ar_chunks_ = (mesh_->mp > 1 && M_ % (4 * 128) == 0) ? 4 : 1;
  if (const char* e = std::getenv("SW_AR_CHUNKS")) {
    const int c = std::atoi(e);
    if (c >= 1 && M_ % c == 0) ar_chunks_ = c;
  }
  {
    // Weight-gradient GEMMs on a side stream: the exposed tail of a fused-AdamW wgrad (its last
    // tiles' optimizer epilogue) overlaps the next dgrad / attention kernel. Measured on the
    // power-capped B200 (LLaMA-7B shape): +1.3% at 8192 tokens per replica, -1.2% at 16384,
    // where the longer K hides that tail anyway and the concurrent kernels cost clock (median
    // 1.15 vs 1.22 GHz). Default: side stream up to 8192 tokens; SW_WGRAD_STREAM=0/1 forces.
    const char* e = std::getenv("SW_WGRAD_STREAM");
    const bool on = e != nullptr ? e[0] != '0' : M_ <= 8192;
    if (on) cuda_check(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking), "cudaStreamCreate");
  }
  for (int i = 0; i < ar_chunks_; ++i) {
    cudaEvent_t a, b;
    cuda_check(cudaEventCreateWithFlags(&a, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventCreateWithFlags(&b, cudaEventDisableTiming), "cudaEventCreate");
    ev_prod_.push_back(a);
    ev_ar_.push_back(b);
  }
}

Model::~Model() {
  if (stream_) cudaStreamSynchronize(stream_);
  if (comm_stream_) cudaStreamSynchronize(comm_stream_);
  if (side_) cudaStreamSynchronize(side_);
  for (cudaEvent_t e : side_ev_) cudaEventDestroy(e);
  if (side_) cudaStreamDestroy(side_);
  for (cudaEvent_t e : events_) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_prod_) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_ar_) cudaEventDestroy(e);
  if (comm_stream_) cudaStreamDestroy(comm_stream_);
  if (dp_stream_) {
    cudaStreamSynchronize(dp_stream_);
    cudaStreamDestroy(dp_stream_);
  }
  for (cudaEvent_t e : dp_ev_) cudaEventDestroy(e);
  if (dec_graph_) cudaGraphExecDestroy(dec_graph_);
  if (dec_out_) cudaFree(dec_out_);
  for (void* p : allocations_) cudaFree(p);
  if (stream_) cudaStreamDestroy(stream_);
}

template <typename T>
T* Model::alloc(int64_t n) {
  void* p = nullptr;
  const size_t bytes = static_cast<size_t>(n > 0 ? n : 1) * sizeof(T);
  cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
  allocations_.push_back(p);
  bytes_ += static_cast<int64_t>(bytes);
  return static_cast<T*>(p);
}

void Model::build_layout() {
  const int t = mesh_->mp;
  const std::vector<NamedShape> shapes = transformer_param_shapes(spec_);
  // init draw bases in tree order (model.hpp:55-68: one stream, 2 draws per normal)
  uint64_t draws = 0;
  std::unordered_map<std::string, std::pair<int, uint64_t>> init_of;
  for (const auto& p : shapes) {
    const std::string leaf = p.name.substr(p.name.rfind('/') + 1);
    if (leaf == "bias") {
      init_of[p.name] = {0, 0};
    } else if (leaf == "scale") {
      init_of[p.name] = {1, 0};
    } else {
      init_of[p.name] = {2, draws};
      draws += 2 * static_cast<uint64_t>(numel_of(p.dims));
    }
  }
  auto make_slot = [&](const NamedShape& p) {
    Slot s;
    s.name = p.name;
    s.global = p.dims;
    const Layout* l = plan_.find(p.name);
    if (l == nullptr) fail(SW_ERR_CONFIG, "ShardingPlan: no entry for parameter '" + p.name + "'");
    s.layout = *l;
    s.local = p.dims;
    s.begin = 0;
    s.end = p.dims.empty() ? 1 : p.dims[0];
    if (l->kind == Layout::kSplit) {
      if (l->dim < 0 || static_cast<size_t>(l->dim) >= p.dims.size()) {
        fail(SW_ERR_PARTITION, "local_shape: split dim " + std::to_string(l->dim) + " out of range for " +
                                   dims_str(p.dims));
      }
      if (p.dims[l->dim] % t != 0) {
        fail(SW_ERR_PARTITION, "local_shape: dim " + std::to_string(l->dim) + " of " + dims_str(p.dims) +
                                   " is not divisible by " + std::to_string(t) + " shards");
      }
      s.local[l->dim] = p.dims[l->dim] / t;
      s.end = s.local[l->dim];  // rank-relative; begin/end rescaled per rank on use
    }
    s.numel = numel_of(s.local);
    s.init = init_of[p.name].first;
    s.draw_base = init_of[p.name].second;
    if (s.init == 2) {
      s.init_scale = p.name.rfind("embed/", 0) == 0 ? 0.02 : 1.0 / std::sqrt(static_cast<double>(p.dims[1]));
    }
    return s;
  };
  std::unordered_map<std::string, const NamedShape*> by_name;
  for (const auto& p : shapes) by_name[p.name] = &p;
  int64_t off = 0;
  auto place = [&](const std::string& name, bool align) {
    const auto it = by_name.find(name);
    Slot s = make_slot(*it->second);
    if (align) off = (off + kAlign - 1) / kAlign * kAlign;
    s.offset = off;
    off += s.numel;
    slots_.push_back(s);
    slot_of_[name] = static_cast<int>(slots_.size()) - 1;
    return static_cast<int>(slots_.size()) - 1;
  };
  // Region 1: the GEMM weight matrices (their wgrad epilogue can apply AdamW in place, see
  // train_step); region 2: embeddings, biases and LayerNorm parameters.
  layers_.resize(L_);
  for (int l = 0; l < L_; ++l) {
    const std::string b = "block_" + std::to_string(l) + "/";
    LayerSlots& ls = layers_[l];
    ls.q_k = place(b + "attn/q/kernel", true);  // q|k|v kernels contiguous: fused [3*d/t, d]
    ls.k_k = place(b + "attn/k/kernel", false);
    ls.v_k = place(b + "attn/v/kernel", false);
    ls.o_k = place(b + "attn/o/kernel", true);
    if (spec_.swiglu) {
      ls.gate_k = place(b + "mlp/fc1/gate/kernel", true);  // gate|up contiguous: fused [2*d_ff/t, d]
      ls.fc1_k = place(b + "mlp/fc1/kernel", false);
    } else {
      ls.fc1_k = place(b + "mlp/fc1/kernel", true);
    }
    ls.fc2_k = place(b + "mlp/fc2/kernel", true);
  }
  layers_end_ = off;
  if (!spec_.tie_embeddings) head_ = place("lm_head/kernel", true);
  weights_end_ = (off + kAlign - 1) / kAlign * kAlign;
  tok_ = place("embed/tok/kernel", true);
  pos_ = place("embed/pos/kernel", true);
  for (int l = 0; l < L_; ++l) {
    const std::string b = "block_" + std::to_string(l) + "/";
    LayerSlots& ls = layers_[l];
    ls.q_b = place(b + "attn/q/bias", true);    // q|k|v biases contiguous: [3*d]
    ls.k_b = place(b + "attn/k/bias", false);
    ls.v_b = place(b + "attn/v/bias", false);
    ls.o_b = place(b + "attn/o/bias", true);
    ls.ln1_s = place(b + "ln1/scale", true);
    if (!spec_.rmsnorm) ls.ln1_b = place(b + "ln1/bias", true);
    ls.ln2_s = place(b + "ln2/scale", true);
    if (!spec_.rmsnorm) ls.ln2_b = place(b + "ln2/bias", true);
    if (!spec_.swiglu) {
      ls.fc1_b = place(b + "mlp/fc1/bias", true);
      ls.fc2_b = place(b + "mlp/fc2/bias", true);
    }
  }
  lnf_s_ = place("final_ln/scale", true);
  if (!spec_.rmsnorm) lnf_b_ = place("final_ln/bias", true);
  flat_n_ = (off + kAlign - 1) / kAlign * kAlign;

  // Which blocks run tensor-parallel: the two sharding rules give column-split QKV / fc1 and
  // row-split O / fc2; a block whose kernels were all degraded to replicated runs replicated.
  auto is_split = [&](int s, int64_t dim) {
    return slots_[s].layout.kind == Layout::kSplit && slots_[s].layout.dim == dim;
  };
  auto is_repl = [&](int s) { return slots_[s].layout.kind == Layout::kReplicated; };
  auto unsupported = [&](const std::string& what) {
    fail(SW_ERR_PARTITION, "GPU executor: unsupported partition for " + what +
                               " (supported: the rule layout or fully replicated)");
  };
  for (const Slot& s : slots_) {
    if (s.global.size() < 2 && !is_repl(static_cast<int>(&s - slots_.data()))) {
      unsupported("1-D parameter '" + s.name + "'");
    }
  }
  if (!is_repl(tok_) || !is_repl(pos_)) unsupported("embedding tables");
  for (int l = 0; l < L_; ++l) {
    const LayerSlots& ls = layers_[l];
    const bool attn_tp = is_split(ls.q_k, 0) && is_split(ls.k_k, 0) && is_split(ls.v_k, 0) && is_split(ls.o_k, 1);
    const bool attn_rep = is_repl(ls.q_k) && is_repl(ls.k_k) && is_repl(ls.v_k) && is_repl(ls.o_k);
    const bool gate_tp = ls.gate_k < 0 || is_split(ls.gate_k, 0);
    const bool gate_rep = ls.gate_k < 0 || is_repl(ls.gate_k);
    const bool mlp_tp = gate_tp && is_split(ls.fc1_k, 0) && is_split(ls.fc2_k, 1);
    const bool mlp_rep = gate_rep && is_repl(ls.fc1_k) && is_repl(ls.fc2_k);
    if (!(attn_tp || attn_rep)) unsupported("the attention kernels of block_" + std::to_string(l));
    if (!(mlp_tp || mlp_rep)) unsupported("the MLP kernels of block_" + std::to_string(l));
    const int ta = attn_tp ? mesh_->mp : 1, tm = mlp_tp ? mesh_->mp : 1;
    if (l == 0) {
      ta_ = ta;
      tm_ = tm;
    } else if (ta != ta_ || tm != tm_) {
      unsupported("blocks with different layouts");
    }
  }
  if (head_ >= 0) {
    if (is_split(head_, 0)) {
      th_ = mesh_->mp;
    } else if (!is_repl(head_)) {
      unsupported("lm_head/kernel");
    }
  }
  if (H_ % ta_ != 0) {
    fail(SW_ERR_PARTITION, "GPU executor: n_heads " + std::to_string(H_) + " not divisible by the " +
                               std::to_string(ta_) + "-way attention split (the reference all-gathers "
                               "q/k/v here, spmd.hpp:58-71)");
  }
  dl_ = d_ / ta_;
  hl_ = H_ / ta_;
  fl_ = dff_ / tm_;
  vl_ = V_ / th_;
  ldv_ = (vl_ + 7) / 8 * 8;
  for (auto [what, v] : {std::pair<const char*, int>{"d_model", d_}, {"d_model/t", dl_}, {"d_ff/t", fl_},
                         {"vocab", vl_}}) {
    if (v % 8 != 0) {
      fail(SW_ERR_CONFIG, std::string("GPU executor: ") + what + " = " + std::to_string(v) +
                              " must be a multiple of 8 (16-byte TMA rows)");
    }
  }
}

void Model::allocate() {
  const int64_t M = M_;
  // Inference-only models (sw_model_create_inference) hold the bf16 GEMM weights, the fp32
  // small parameters (region 2) and, per layer, only the K/V cache (the qkv activations): no
  // fp32 master copies of the GEMM weights, no gradients or AdamW moments, and the other
  // activations alternate between two buffers because nothing reads them back.
  const int64_t n_small = flat_n_ - weights_end_;
  const int keep = inference_ ? std::min(L_, 2) : L_;  // distinct per-layer activation buffers
  for (int dev : mesh_->local_devices()) {
    Rank R;
    R.device = dev;
    R.dpi = mesh_->dp_index(dev);
    R.mpi = mesh_->mp_index(dev);
    R.w = alloc<bf16>(flat_n_);
    cuda_check(cudaMemsetAsync(R.w, 0, flat_n_ * 2, stream_), "memset");
    if (inference_) {
      float* small = alloc<float>(n_small);
      cuda_check(cudaMemsetAsync(small, 0, n_small * 4, stream_), "memset");
      R.p_small = small;
    } else {
      R.p = alloc<float>(flat_n_);
      R.g = alloc<float>(flat_n_);
      R.m = alloc<float>(flat_n_);
      R.v = alloc<float>(flat_n_);
      cuda_check(cudaMemsetAsync(R.p, 0, flat_n_ * 4, stream_), "memset");
      cuda_check(cudaMemsetAsync(R.g, 0, flat_n_ * 4, stream_), "memset");
      cuda_check(cudaMemsetAsync(R.m, 0, flat_n_ * 4, stream_), "memset");
      cuda_check(cudaMemsetAsync(R.v, 0, flat_n_ * 4, stream_), "memset");
    }
    for (int l = 0; l <= L_; ++l) R.hs.push_back(l <= keep ? alloc<float>(M * d_) : R.hs[l % 2]);
    for (int l = 0; l < L_; ++l) {
      R.qkv.push_back(alloc<bf16>(M * 3 * dl_));
      if (l >= keep) {
        const int j = l % 2;
        R.hmid.push_back(R.hmid[j]);
        R.stats1.push_back(R.stats1[j]);
        R.stats2.push_back(R.stats2[j]);
        R.a1.push_back(R.a1[j]);
        R.a2.push_back(R.a2[j]);
        R.o.push_back(R.o[j]);
        R.lse.push_back(R.lse[j]);
        R.pre.push_back(R.pre[j]);
        R.act.push_back(R.act[j]);
        continue;
      }
      R.hmid.push_back(alloc<float>(M * d_));
      R.stats1.push_back(alloc<float>(2 * M));
      R.stats2.push_back(alloc<float>(2 * M));
      R.a1.push_back(alloc<bf16>(M * d_));
      R.a2.push_back(alloc<bf16>(M * d_));
      R.o.push_back(alloc<bf16>(M * dl_));
      R.lse.push_back(alloc<float>(M * hl_));
      R.pre.push_back(alloc<bf16>(M * fl_ * (spec_.swiglu ? 2 : 1)));  // SwiGLU: gate | up
      R.act.push_back(alloc<bf16>(M * fl_));
    }
    R.statsf = alloc<float>(2 * M);
    R.f = alloc<bf16>(M * d_);
    R.logits = alloc<bf16>(M * ldv_);
    R.tokens = alloc<int32_t>(M);
    R.targets = alloc<int32_t>(M);
    R.weights = alloc<float>(M);
    R.wloss = alloc<float>(M);
    R.wsum = alloc<float>(1);
    R.loss = alloc<double>(1);
    R.part = alloc<float>(M * d_);
    if (ar_bf16_) R.arb = alloc<bf16>(M * d_);
    R.xstats = alloc<float>(static_cast<int64_t>(mesh_->mp) * M * 2);
    R.xt = alloc<float>(M);
    R.xlse = alloc<float>(M);
    if (!inference_) {  // backward-only buffers
      R.dx = alloc<float>(M * d_);
      R.gres = alloc<float>(M * d_);
      R.gb = alloc<bf16>(M * d_);
      R.dpre = alloc<bf16>(M * fl_ * (spec_.swiglu ? 2 : 1));
      R.dout = alloc<bf16>(M * dl_);
      R.dqkv = alloc<bf16>(M * 3 * dl_);
      const int64_t chunks = (M + 255) / 256;
      int64_t widest = d_;
      if (3 * dl_ > widest) widest = 3 * dl_;
      if (fl_ > widest) widest = fl_;
      // also holds the GeLU-backward epilogue's per-32-row partial column sums of dpre
      R.col_scratch = alloc<float>(std::max(chunks * widest, ((M + 31) / 32) * std::max<int64_t>(fl_, 3 * dl_)));
      R.ln_partials = alloc<float>(k::layernorm_bwd_partials(d_));
      R.tok_keys = alloc<uint32_t>(k::embed_bwd_keys(M_));
      R.attn_scratch = alloc<float>(std::max<int64_t>(M * hl_ + M * 2 * dl_ + 64,
                                                      k::attention_bwd_scratch_floats(B_, T_, hl_, hd_)));
    }
    ranks_.push_back(R);
  }
  d_flag_ = alloc<int>(1);
  cuda_check(cudaStreamSynchronize(stream_), "allocate");
}

std::vector<Rank*> Model::replica(int dpi) {
  std::vector<Rank*> g;
  for (Rank& R : ranks_) {
    if (R.dpi == dpi) g.push_back(&R);
  }
  return g;
}

// ---------------------------------------------------------------------------------------------
// parameters
// ---------------------------------------------------------------------------------------------
void Model::init_params(uint64_t seed, const std::string& stream_name) {
  const uint64_t key = mix64(seed ^ mix64(fnv1a(stream_name)));
  // inference-only: a GEMM weight is drawn in fp32 into a scratch slot and rounded into w
  float* scratch = nullptr;
  if (inference_) {
    int64_t widest = 0;
    for (const Slot& s : slots_)
      if (s.offset < weights_end_) widest = std::max(widest, s.numel);
    if (widest > 0) cuda_check(cudaMalloc(&scratch, widest * 4), "cudaMalloc");
  }
  for (Rank& R : ranks_) {
    for (const Slot& s : slots_) {
      const bool via_scratch = inference_ && s.offset < weights_end_;
      float* dst = via_scratch ? scratch : pval(R, s.offset);
      if (s.init == 0) {
        cuda_check(cudaMemsetAsync(dst, 0, s.numel * 4, stream_), "memset");
      } else if (s.init == 1) {
        k::fill_f32(dst, s.numel, 1.0f, stream_);
        ++launches_;
      } else {
        int64_t r0 = 0, c0 = 0;
        if (s.layout.kind == Layout::kSplit) {
          (s.layout.dim == 0 ? r0 : c0) = s.local[s.layout.dim] * R.mpi;
        }
        k::init_normal(dst, s.local[0], s.local[1], r0, c0, s.global[1], key, s.draw_base,
                       s.init_scale, stream_);
        ++launches_;
      }
      if (via_scratch) {
        k::cast_f32_bf16(scratch, W(R, static_cast<int>(&s - slots_.data())), s.numel, stream_);
        ++launches_;
      }
    }
    if (inference_) {
      k::cast_f32_bf16(R.p_small, R.w + weights_end_, flat_n_ - weights_end_, stream_);
    } else {
      cuda_check(cudaMemsetAsync(R.m, 0, flat_n_ * 4, stream_), "memset");
      cuda_check(cudaMemsetAsync(R.v, 0, flat_n_ * 4, stream_), "memset");
      k::cast_f32_bf16(R.p, R.w, flat_n_, stream_);
    }
    ++launches_;
  }
  if (scratch != nullptr) {
    cuda_check(cudaStreamSynchronize(stream_), "init_params");
    cudaFree(scratch);
  }
  step_ = 0;
  seed_ = seed;
  poisoned_ = false;
  cuda_check(cudaGetLastError(), "init_params");
}

void Model::set_param(const std::string& name, const float* full, int64_t numel) {
  set_tensor(name, 0, full, numel);
}

void Model::set_tensor(const std::string& name, int which, const float* full, int64_t numel) {
  const auto it = slot_of_.find(name);
  if (it == slot_of_.end()) fail(SW_ERR_CONFIG, "TrainState: no parameter named '" + name + "'");
  const Slot& s = slots_[it->second];
  if (numel != numel_of(s.global)) {
    fail(SW_ERR_SHAPE, "set_param: '" + name + "' expects " + std::to_string(numel_of(s.global)) +
                           " elements, got " + std::to_string(numel));
  }
  if (which != 0 && which != 2 && which != 3) fail(SW_ERR_CONFIG, "set_tensor: `which` must be 0, 2 or 3");
  if (which != 0) check_trainable("set_tensor (AdamW moments)");
  const bool via_scratch = inference_ && s.offset < weights_end_;
  float* scratch = nullptr;
  if (via_scratch) cuda_check(cudaMalloc(&scratch, s.numel * 4), "cudaMalloc");
  for (Rank& R : ranks_) {
    float* dst = via_scratch ? scratch : which == 0 ? pval(R, s.offset) : (which == 2 ? R.m : R.v) + s.offset;
    if (s.layout.kind != Layout::kSplit) {
      cuda_check(cudaMemcpyAsync(dst, full, numel * 4, cudaMemcpyHostToDevice, stream_), "H2D");
    } else {
      const int64_t rows = s.global[0], cols = s.global[1];
      if (s.layout.dim == 0) {
        const int64_t lr = s.local[0];
        cuda_check(cudaMemcpyAsync(dst, full + R.mpi * lr * cols, lr * cols * 4, cudaMemcpyHostToDevice, stream_),
                   "H2D");
      } else {
        const int64_t lc = s.local[1];
        cuda_check(cudaMemcpy2DAsync(dst, lc * 4, full + R.mpi * lc, cols * 4, lc * 4, rows,
                                     cudaMemcpyHostToDevice, stream_),
                   "H2D 2D");
      }
    }
    if (which == 0) k::cast_f32_bf16(dst, R.w + s.offset, s.numel, stream_);
    if (via_scratch) cuda_check(cudaStreamSynchronize(stream_), "set_param");  // scratch reused per rank
  }
  cuda_check(cudaStreamSynchronize(stream_), "set_param");
  if (scratch != nullptr) cudaFree(scratch);
}

void Model::save_checkpoint(const std::string& path, const std::vector<CkptRng>& rngs) {
  check_trainable("save_checkpoint");
  check_not_poisoned("save_checkpoint");
  Checkpoint ck;
  ck.step = step_;
  ck.seed = seed_;
  ck.rngs = rngs;
  static const char* kPrefix[3] = {"params/", "adam_m/", "adam_v/"};
  static const int kWhich[3] = {0, 2, 3};
  for (const NamedShape& ns : transformer_param_shapes(spec_)) {  // tree order (model.hpp:17-43)
    int64_t n = 1;
    for (int64_t dd : ns.dims) n *= dd;
    for (int i = 0; i < 3; ++i) {
      CkptRecord rec;
      rec.name = std::string(kPrefix[i]) + ns.name;
      rec.shape.assign(ns.dims.begin(), ns.dims.end());
      rec.data.resize(static_cast<size_t>(n));
      get_tensor(ns.name, kWhich[i], rec.data.data(), n);  // collective over the mp group under NCCL
      ck.records.push_back(std::move(rec));
    }
  }
  // one writer per job: the emulated mesh's process, or world rank 0
  if (mesh_->emulated || mesh_->rank == 0) write_checkpoint(path, ck);
}

void Model::load_checkpoint(const std::string& path) {
  Checkpoint ck = read_checkpoint(path);
  std::unordered_map<std::string, size_t> in_file;
  for (size_t r = 0; r < ck.records.size(); r += 3) in_file[ck.records[r].name.substr(7)] = r;
  for (const NamedShape& ns : transformer_param_shapes(spec_)) {
    const auto f = in_file.find(ns.name);
    if (f == in_file.end()) {
      fail(SW_ERR_CHECKPOINT, "checkpoint: no record for parameter '" + ns.name + "' of this model");
    }
    const std::vector<int64_t> want(ns.dims.begin(), ns.dims.end());
    if (ck.records[f->second].shape != want) {
      fail(SW_ERR_CHECKPOINT, "checkpoint: record 'params/" + ns.name + "' does not match the model's shape");
    }
  }
  if (in_file.size() != slot_of_.size()) {
    for (const auto& kv : in_file) {
      if (slot_of_.find(kv.first) == slot_of_.end()) {
        fail(SW_ERR_CHECKPOINT, "checkpoint: record 'params/" + kv.first + "' names no parameter of this model");
      }
    }
  }
  for (size_t r = 0; r < ck.records.size(); r += 3) {
    const std::string name = ck.records[r].name.substr(7);
    const int64_t n = static_cast<int64_t>(ck.records[r].data.size());
    set_tensor(name, 0, ck.records[r].data.data(), n);
    if (inference_) continue;  // the Predictor's load: parameters only
    set_tensor(name, 2, ck.records[r + 1].data.data(), n);
    set_tensor(name, 3, ck.records[r + 2].data.data(), n);
  }
  step_ = ck.step;
  seed_ = ck.seed;
  loaded_rngs_ = std::move(ck.rngs);
  poisoned_ = false;
}

void Model::get_tensor(const std::string& name, int which, float* full, int64_t numel) {
  const auto it = slot_of_.find(name);
  if (it == slot_of_.end()) fail(SW_ERR_CONFIG, "TrainState: no parameter named '" + name + "'");
  const Slot& s = slots_[it->second];
  if (numel != numel_of(s.global)) {
    fail(SW_ERR_SHAPE, "get_tensor: '" + name + "' has " + std::to_string(numel_of(s.global)) +
                           " elements, got a buffer of " + std::to_string(numel));
  }
  if (which < 0 || which > 3) fail(SW_ERR_CONFIG, "get_tensor: `which` must be 0..3");
  if (which != 0) check_trainable("get_tensor (gradients / AdamW moments)");
  // an inference-only model keeps GEMM weights in bf16 only: they are widened into scratch
  struct Scratch {
    float* p = nullptr;
    ~Scratch() {
      if (p != nullptr) cudaFree(p);
    }
  } scratch;
  const bool widen = inference_ && s.offset < weights_end_;
  if (widen) cuda_check(cudaMalloc(&scratch.p, s.numel * 4), "cudaMalloc");
  auto src = [&](Rank& R) -> const float* {
    if (widen) {
      k::cast_bf16_f32(R.w + s.offset, scratch.p, s.numel, stream_);
      cuda_check(cudaStreamSynchronize(stream_), "get_tensor");
      return scratch.p;
    }
    if (which == 0) return pval(R, s.offset);
    return (which == 1 ? R.g : which == 2 ? R.m : R.v) + s.offset;
  };
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  if (s.layout.kind != Layout::kSplit) {
    Rank& R = *replica(mesh_->emulated ? 0 : ranks_[0].dpi)[0];
    cuda_check(cudaMemcpy(full, src(R), numel * 4, cudaMemcpyDeviceToHost), "D2H");
    return;
  }
  const int64_t rows = s.global[0], cols = s.global[1];
  if (mesh_->emulated) {
    for (Rank* R : replica(0)) {
      const float* from = src(*R);
      if (s.layout.dim == 0) {
        cuda_check(cudaMemcpy(full + R->mpi * s.local[0] * cols, from, s.numel * 4, cudaMemcpyDeviceToHost), "D2H");
      } else {
        const int64_t lc = s.local[1];
        cuda_check(cudaMemcpy2D(full + R->mpi * lc, cols * 4, from, lc * 4, lc * 4, rows, cudaMemcpyDeviceToHost),
                   "D2H 2D");
      }
    }
    return;
  }
  // NCCL mode: all-gather the shards of this replica's mp group (collective over mp ranks).
  Rank& R = ranks_[0];
  float* tmp = nullptr;
  cuda_check(cudaMalloc(&tmp, numel * 4), "cudaMalloc");
  nccl_check(ncclAllGather(src(R), tmp, s.numel, ncclFloat, mesh_->mp_comm, stream_), "AllGather");
  std::vector<float> host(numel);
  cuda_check(cudaMemcpyAsync(host.data(), tmp, numel * 4, cudaMemcpyDeviceToHost, stream_), "D2H");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  cudaFree(tmp);
  const int t = mesh_->mp;
  if (s.layout.dim == 0) {
    std::memcpy(full, host.data(), numel * 4);
  } else {
    const int64_t lc = s.local[1];
    for (int r = 0; r < t; ++r)
      for (int64_t i = 0; i < rows; ++i)
        std::memcpy(full + i * cols + r * lc, host.data() + r * s.numel + i * lc, lc * 4);
  }
}

void Model::stage_batch(const int32_t* tokens, const int32_t* targets, const float* weights) {
  for (Rank& R : ranks_) {
    const int64_t off = static_cast<int64_t>(R.dpi) * M_;
    cuda_check(cudaMemcpyAsync(R.tokens, tokens + off, M_ * 4, cudaMemcpyHostToDevice, stream_), "H2D");
    cuda_check(cudaMemcpyAsync(R.targets, targets + off, M_ * 4, cudaMemcpyHostToDevice, stream_), "H2D");
    if (weights != nullptr) {
      cuda_check(cudaMemcpyAsync(R.weights, weights + off, M_ * 4, cudaMemcpyHostToDevice, stream_), "H2D");
    } else {
      k::fill_f32(R.weights, M_, 1.0f, stream_);
      ++launches_;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// collectives
// ---------------------------------------------------------------------------------------------
void Model::ar_mp_ptrs(std::vector<Rank*>& grp, const std::vector<float*>& ptrs, int64_t n, cudaStream_t s) {
  if (mesh_->mp == 1) return;
  if (s == nullptr) s = stream_;
  const double t = mesh_->mp;
  tic(s);
  if (mesh_->emulated) {
    k::sum_ranks_f32(ptrs.data(), static_cast<int>(ptrs.size()), n, 1.0f, s);
    ++launches_;
  } else {
    nccl_check(ncclAllReduce(ptrs[0], ptrs[0], n, ncclFloat, ncclSum, mesh_->mp_comm, s), "AllReduce");
  }
  toc(kProfComm, 2.0 * (t - 1) / t * 4.0 * n, s);  // NCCL bus bytes
  mesh_->record(CollKind::kAllReduce, mesh_->mp_group(grp[0]->dpi), static_cast<uint64_t>(n) * 4);
}

void Model::ar_mp_ptrs(std::vector<Rank*>& grp, const std::vector<bf16*>& ptrs, int64_t n, cudaStream_t s) {
  if (mesh_->mp == 1) return;
  const double t = mesh_->mp;
  tic(s);
  if (mesh_->emulated) {
    k::sum_ranks_bf16(ptrs.data(), static_cast<int>(ptrs.size()), n, 1.0f, s);
    ++launches_;
  } else {
    nccl_check(ncclAllReduce(ptrs[0], ptrs[0], n, ncclBfloat16, ncclSum, mesh_->mp_comm, s), "AllReduce(bf16)");
  }
  toc(kProfComm, 2.0 * (t - 1) / t * 2.0 * n, s);  // NCCL bus bytes
  mesh_->record(CollKind::kAllReduce, mesh_->mp_group(grp[0]->dpi), static_cast<uint64_t>(n) * 2);
}

void Model::row_parallel_ar(std::vector<Rank*>& grp, bf16* Rank::*buf, int width, const RowFn& produce,
                            const RowFn& consume) {
  const int C = ar_chunks_;
  const int64_t rows = M_ / C;
  for (int c = 0; c < C; ++c) {
    for (Rank* R : grp) produce(*R, c * rows, rows);
    cuda_check(cudaEventRecord(ev_prod_[c], stream_), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(comm_stream_, ev_prod_[c], 0), "cudaStreamWaitEvent");
    std::vector<bf16*> ptrs;
    for (Rank* R : grp) ptrs.push_back(R->*buf + c * rows * width);
    ar_mp_ptrs(grp, ptrs, rows * width, comm_stream_);
    cuda_check(cudaEventRecord(ev_ar_[c], comm_stream_), "cudaEventRecord");
  }
  for (int c = 0; c < C; ++c) {
    cuda_check(cudaStreamWaitEvent(stream_, ev_ar_[c], 0), "cudaStreamWaitEvent");
    for (Rank* R : grp) consume(*R, c * rows, rows);
  }
}

void Model::row_ar(std::vector<Rank*>& grp, float* Rank::*f32buf, const std::function<const bf16*(Rank&)>& a,
                   int64_t lda, int K, int w_slot, int b_mn, const ConsFn& consume) {
  const int d = d_;
  const int64_t ldb = b_mn ? d : K;
  if (ar_bf16_) {
    row_parallel_ar(
        grp, &Rank::arb, d,
        [&](Rank& R, int64_t r0, int64_t rows) {
          gemm(R, static_cast<int>(rows), d, K, a(R) + r0 * lda, lda, 0, W(R, w_slot), ldb, b_mn,
               static_cast<int>(Epi::kStoreBf16), R.arb + r0 * d, d);
        },
        [&](Rank& R, int64_t r0, int64_t rows) { consume(R, r0, rows, nullptr, R.arb + r0 * d); });
  } else {
    row_parallel_ar(
        grp, f32buf, d,
        [&](Rank& R, int64_t r0, int64_t rows) {
          gemm(R, static_cast<int>(rows), d, K, a(R) + r0 * lda, lda, 0, W(R, w_slot), ldb, b_mn,
               static_cast<int>(Epi::kStoreF32), R.*f32buf + r0 * d, d);
        },
        [&](Rank& R, int64_t r0, int64_t rows) { consume(R, r0, rows, R.*f32buf + r0 * d, nullptr); });
  }
}

void Model::row_parallel_ar(std::vector<Rank*>& grp, float* Rank::*buf, int width, const RowFn& produce,
                            const RowFn& consume) {
  const int C = ar_chunks_;
  const int64_t rows = M_ / C;
  for (int c = 0; c < C; ++c) {
    for (Rank* R : grp) produce(*R, c * rows, rows);
    cuda_check(cudaEventRecord(ev_prod_[c], stream_), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(comm_stream_, ev_prod_[c], 0), "cudaStreamWaitEvent");
    std::vector<float*> ptrs;
    for (Rank* R : grp) ptrs.push_back(R->*buf + c * rows * width);
    ar_mp_ptrs(grp, ptrs, rows * width, comm_stream_);
    cuda_check(cudaEventRecord(ev_ar_[c], comm_stream_), "cudaEventRecord");
  }
  for (int c = 0; c < C; ++c) {
    cuda_check(cudaStreamWaitEvent(stream_, ev_ar_[c], 0), "cudaStreamWaitEvent");
    for (Rank* R : grp) consume(*R, c * rows, rows);
  }
}

void Model::ar_mp(std::vector<Rank*>& grp, float* Rank::*buf, int64_t n) {
  std::vector<float*> ptrs;
  for (Rank* R : grp) ptrs.push_back(R->*buf);
  ar_mp_ptrs(grp, ptrs, n);
}

// In-place all-gather of a replicated 1-D slot's grad whose chunk `mpi` was produced locally.
void Model::ag_mp_slot(std::vector<Rank*>& grp, int slot, int64_t chunk) {
  if (mesh_->mp == 1) return;
  const int t = mesh_->mp;
  if (mesh_->emulated) {
    for (Rank* src : grp) {
      for (Rank* dst : grp) {
        if (dst == src) continue;
        cuda_check(cudaMemcpyAsync(G(*dst, slot) + src->mpi * chunk, G(*src, slot) + src->mpi * chunk,
                                   chunk * 4, cudaMemcpyDeviceToDevice, stream_),
                   "D2D");
      }
    }
  } else {
    Rank& R = *grp[0];
    float* base = G(R, slot);
    nccl_check(ncclAllGather(base + R.mpi * chunk, base, chunk, ncclFloat, mesh_->mp_comm, stream_), "AllGather");
  }
  mesh_->record(CollKind::kAllGather, mesh_->mp_group(grp[0]->dpi), static_cast<uint64_t>(chunk) * t * 4);
}

void Model::ag_mp_buf(std::vector<Rank*>& grp, float* Rank::*buf, int64_t chunk) {
  if (mesh_->mp == 1) return;
  const int t = mesh_->mp;
  if (mesh_->emulated) {
    for (Rank* src : grp) {
      for (Rank* dst : grp) {
        if (dst == src) continue;
        cuda_check(cudaMemcpyAsync(dst->*buf + src->mpi * chunk, src->*buf + src->mpi * chunk, chunk * 4,
                                   cudaMemcpyDeviceToDevice, stream_),
                   "D2D");
      }
    }
  } else {
    Rank& R = *grp[0];
    nccl_check(ncclAllGather(R.*buf + R.mpi * chunk, R.*buf, chunk, ncclFloat, mesh_->mp_comm, stream_),
               "AllGather");
  }
  mesh_->record(CollKind::kAllGather, mesh_->mp_group(grp[0]->dpi), static_cast<uint64_t>(chunk) * t * 4);
}

void Model::gemm(Rank& R, int M, int N, int K, const void* A, int64_t lda, int a_mn, const void* B,
                 int64_t ldb, int b_mn, int epi, void* C, int64_t ldc, void* C2, int64_t ldc2,
                 const float* bias, const void* aux, int64_t ld_aux, int accumulate, int bias_seg,
                 int64_t bias_seg_stride, int swiglu_half, float* delta, int delta_T, float* colsum) {
  (void)R;
  GemmParams p;
  p.colsum = colsum;
  p.delta = delta;
  p.delta_T = delta_T;
  p.swiglu_half = swiglu_half;
  p.M = M;
  p.N = N;
  p.K = K;
  p.A = A;
  p.lda = lda;
  p.a_mn_major = a_mn;
  p.B = B;
  p.ldb = ldb;
  p.b_mn_major = b_mn;
  p.epi = static_cast<Epi>(epi);
  p.C = C;
  p.ldc = ldc;
  p.C2 = C2;
  p.ldc2 = ldc2;
  p.bias = bias;
  p.bias_seg = bias_seg;
  p.bias_seg_stride = bias_seg_stride;
  p.aux = aux;
  p.ld_aux = ld_aux;
  p.accumulate = accumulate;
  p.pdl = prof_ ? 0 : pdl_;
  tic();
  cuda_check(gemm_bf16(p, stream_), "gemm launch");
  // kSwiGLU multiplies by the fused [gate; up] weight: 2N output columns of MMA work
  toc(kProfGemm, 2.0 * M * (epi == static_cast<int>(Epi::kSwiGLU) ? 2.0 * N : N) * static_cast<double>(K));
  if (prof_) {
    prof_tag_.resize(prof_rec_.size());
    prof_tag_.back() = "gemm," + std::to_string(M) + "," + std::to_string(N) + "," + std::to_string(K) + ",epi" +
                       std::to_string(epi) + (a_mn ? ",A_mn" : ",A_k") + (b_mn ? ",B_mn" : ",B_k");
  }
  ++launches_;
}

bool Model::gemm_dout(Rank& R, int l, const bf16* wo) {
  static const bool fuse = [] {
    const char* e = std::getenv("SW_FUSE_DELTA");
    return e == nullptr || std::atoi(e) != 0;
  }();
  const int M = static_cast<int>(M_);
  if (fuse && hd_ == 128) {
    GemmParams p;
    p.M = M;
    p.N = dl_;
    p.K = d_;
    p.b_mn_major = 1;
    p.ldc = dl_;
    p.aux = R.o[l];
    p.ld_aux = dl_;
    p.delta = R.attn_scratch;
    p.delta_T = T_;
    if (gemm_delta_ok(p)) {
      gemm(R, M, dl_, d_, R.gb, d_, 0, wo, dl_, 1, static_cast<int>(Epi::kBf16Delta), R.dout, dl_, nullptr, 0,
           nullptr, R.o[l], dl_, 0, 0, 0, 0, R.attn_scratch, T_);
      return true;
    }
  }
  gemm(R, M, dl_, d_, R.gb, d_, 0, wo, dl_, 1, static_cast<int>(Epi::kStoreBf16), R.dout, dl_);
  return false;
}

// ---------------------------------------------------------------------------------------------
// forward (transformer_logits + transformer_loss, model.hpp:76-152)
// ---------------------------------------------------------------------------------------------
void Model::forward_replica(std::vector<Rank*>& grp, bool need_grad) {
  const int64_t M = M_;
  const int d = d_, dl = dl_, fl = fl_;
  for (Rank* R : grp) {
    k::embed_fwd(R->tokens, P(*R, tok_), P(*R, pos_), R->hs[0], M, T_, d, stream_);
    ++launches_;
  }
  for (int l = 0; l < L_; ++l) {
    const LayerSlots& ls = layers_[l];
    for (Rank* R : grp) {
      tic();
      k::layernorm_fwd(R->hs[l], P(*R, ls.ln1_s), Pn(*R, ls.ln1_b), R->a1[l], R->stats1[l], R->stats1[l] + M,
                       M, d, 1e-5f, stream_, spec_.rmsnorm);
      toc(kProfNorm, 6.0 * M * d);
      ++launches_;
      // column-parallel QKV (spmd.hpp:284-303): [M, d] x [3*dl, d]^T, bias slices of q|k|v
      gemm(*R, static_cast<int>(M), 3 * dl, d, R->a1[l], d, 0, W(*R, ls.q_k), d, 0,
           static_cast<int>(Epi::kStoreBf16), R->qkv[l], 3 * dl, nullptr, 0, P(*R, ls.q_b) + R->mpi * dl,
           nullptr, 0, 0, dl, d);
      tic();
      k::attention_fwd(R->qkv[l], R->o[l], R->lse[l], B_, T_, hl_, hd_, stream_);
      toc(kProfAttnFwd, 2.0 * B_ * hl_ * static_cast<double>(T_) * T_ * hd_);
      ++launches_;
    }
    // row-parallel O (spmd.hpp:305-324): local GEMM, all-reduce, then + bias (+ residual)
    if (ta_ == 1) {
      for (Rank* R : grp) {
        gemm(*R, static_cast<int>(M), d, dl, R->o[l], dl, 0, W(*R, ls.o_k), dl, 0,
             static_cast<int>(Epi::kResidF32), R->hmid[l], d, nullptr, 0, P(*R, ls.o_b), R->hs[l], d);
      }
    } else {
      row_ar(
          grp, &Rank::part, [&](Rank& R) -> const bf16* { return R.o[l]; }, dl, dl, ls.o_k, 0,
          [&](Rank& R, int64_t r0, int64_t rows, const float* f32, const bf16* b16) {
            if (b16 != nullptr)
              k::add_residual_bias(R.hs[l] + r0 * d, b16, P(R, ls.o_b), R.hmid[l] + r0 * d, rows, d, stream_);
            else
              k::add_residual_bias(R.hs[l] + r0 * d, f32, P(R, ls.o_b), R.hmid[l] + r0 * d, rows, d, stream_);
            ++launches_;
          });
    }
    for (Rank* R : grp) {
      tic();
      k::layernorm_fwd(R->hmid[l], P(*R, ls.ln2_s), Pn(*R, ls.ln2_b), R->a2[l], R->stats2[l], R->stats2[l] + M,
                       M, d, 1e-5f, stream_, spec_.rmsnorm);
      toc(kProfNorm, 6.0 * M * d);
      ++launches_;
      if (spec_.swiglu) {
        // one GEMM for gate and up: h = silu(x W_g^T) * (x W_u^T), pre = gate | up (bf16)
        gemm(*R, static_cast<int>(M), fl, d, R->a2[l], d, 0, W(*R, ls.gate_k), d, 0,
             static_cast<int>(Epi::kSwiGLU), R->act[l], fl, R->pre[l], 2 * fl, nullptr, nullptr, 0, 0, 0, 0, fl);
      } else {
        gemm(*R, static_cast<int>(M), fl, d, R->a2[l], d, 0, W(*R, ls.fc1_k), d, 0,
             static_cast<int>(Epi::kBiasGelu), R->pre[l], fl, R->act[l], fl, P(*R, ls.fc1_b) + R->mpi * fl);
      }
    }
    if (tm_ == 1) {
      for (Rank* R : grp) {
        gemm(*R, static_cast<int>(M), d, fl, R->act[l], fl, 0, W(*R, ls.fc2_k), fl, 0,
             static_cast<int>(Epi::kResidF32), R->hs[l + 1], d, nullptr, 0, Pn(*R, ls.fc2_b), R->hmid[l], d);
      }
    } else {
      row_ar(
          grp, &Rank::part, [&](Rank& R) -> const bf16* { return R.act[l]; }, fl, fl, ls.fc2_k, 0,
          [&](Rank& R, int64_t r0, int64_t rows, const float* f32, const bf16* b16) {
            if (b16 != nullptr)
              k::add_residual_bias(R.hmid[l] + r0 * d, b16, Pn(R, ls.fc2_b), R.hs[l + 1] + r0 * d, rows, d,
                                   stream_);
            else
              k::add_residual_bias(R.hmid[l] + r0 * d, f32, Pn(R, ls.fc2_b), R.hs[l + 1] + r0 * d, rows, d,
                                   stream_);
            ++launches_;
          });
    }
  }
  const int head = head_ >= 0 ? head_ : tok_;
  static const bool head_row_on = [] {
    const char* e = std::getenv("SW_PREFILL_HEAD_ROW");
    return !(e != nullptr && e[0] == '0');
  }();
  if (head_row_ >= 0 && !head_row_on) {  // all rows through the head, then the rows picked
    for (Rank* R : grp) {
      DecodeBufs& D = dec_[static_cast<size_t>(R - ranks_.data())];
      k::layernorm_fwd(R->hs[L_], P(*R, lnf_s_), Pn(*R, lnf_b_), R->f, R->statsf, R->statsf + M, M, d, 1e-5f,
                       stream_, spec_.rmsnorm);
      gemm(*R, static_cast<int>(M), vl_, d, R->f, d, 0, W(*R, head), d, 0, static_cast<int>(Epi::kStoreBf16),
           R->logits, ldv_);
      cuda_check(cudaMemcpy2DAsync(D.logits + static_cast<int64_t>(head_seq_) * ldv_, static_cast<size_t>(ldv_) * 2,
                                   R->logits + static_cast<int64_t>(head_row_) * ldv_,
                                   static_cast<size_t>(T_) * ldv_ * 2, static_cast<size_t>(ldv_) * 2, B_,
                                   cudaMemcpyDeviceToDevice, stream_),
                 "D2D 2D");
    }
    return;
  }
  if (head_row_ >= 0) {
    // prefill: only row head_row_ of every sequence needs logits (the next token); its final
    // hidden row goes through the head as a small-M GEMM into the decode buffers, no loss
    for (Rank* R : grp) {
      DecodeBufs& D = dec_[static_cast<size_t>(R - ranks_.data())];
      k::layernorm_fwd(R->hs[L_], P(*R, lnf_s_), Pn(*R, lnf_b_), R->f, R->statsf, R->statsf + M, M, d, 1e-5f,
                       stream_, spec_.rmsnorm);
      ++launches_;
      bf16* f = D.f + static_cast<int64_t>(head_seq_) * d;
      cuda_check(cudaMemcpy2DAsync(f, static_cast<size_t>(d) * 2, R->f + static_cast<int64_t>(head_row_) * d,
                                   static_cast<size_t>(T_) * d * 2, static_cast<size_t>(d) * 2, B_,
                                   cudaMemcpyDeviceToDevice, stream_),
                 "D2D 2D");
      gemm(*R, B_, vl_, d, f, d, 0, W(*R, head), d, 0, static_cast<int>(Epi::kStoreBf16),
           D.logits + static_cast<int64_t>(head_seq_) * ldv_, ldv_);
    }
    return;
  }
  for (Rank* R : grp) {
    tic();
    k::layernorm_fwd(R->hs[L_], P(*R, lnf_s_), Pn(*R, lnf_b_), R->f, R->statsf, R->statsf + M, M, d, 1e-5f,
                     stream_, spec_.rmsnorm);
    toc(kProfNorm, 6.0 * M * d);
    ++launches_;
    // LM head (replicated under the reference plan: every rank computes all V columns)
    gemm(*R, static_cast<int>(M), vl_, d, R->f, d, 0, W(*R, head), d, 0, static_cast<int>(Epi::kStoreBf16),
         R->logits, ldv_);
    k::sum_f32(R->weights, M, R->wsum, stream_);
    ++launches_;
  }
  if (th_ == 1) {
    for (Rank* R : grp) {
      tic();
      k::xent_fwd_bwd(R->logits, ldv_, M, vl_, R->targets, R->weights, R->wsum, R->wloss, need_grad ? 1 : 0,
                      stream_);
      toc(kProfXent, (need_grad ? 4.0 : 2.0) * M * vl_);
      ++launches_;
    }
  } else {
    // vocab-parallel CE: local (max, sumexp) + owned target logit, exchanged across the mp group
    for (Rank* R : grp) {
      tic();
      k::xent_vp_stats(R->logits, ldv_, M, vl_, R->mpi * vl_, R->targets, R->xstats + R->mpi * M * 2, R->xt,
                       stream_);
      toc(kProfXent, 2.0 * M * vl_);
      ++launches_;
    }
    ag_mp_buf(grp, &Rank::xstats, M * 2);
    ar_mp(grp, &Rank::xt, M);
    for (Rank* R : grp) {
      k::xent_vp_combine(R->xstats, mesh_->mp, M, R->xt, R->weights, R->xlse, R->wloss, stream_);
      ++launches_;
      if (need_grad) {
        tic();
        k::xent_vp_grad(R->logits, ldv_, M, vl_, R->mpi * vl_, R->targets, R->xlse, R->weights, R->wsum, stream_);
        toc(kProfXent, 4.0 * M * vl_);
        ++launches_;
      }
    }
  }
  for (Rank* R : grp) {
    k::loss_reduce(R->wloss, M, R->wsum, R->loss, stream_, fused_ != nullptr ? d_flag_ : nullptr);
    ++launches_;
  }
}

// ---------------------------------------------------------------------------------------------
// backward (the VJPs of autodiff.hpp, executed with the partition rules of spmd.hpp:342-387)
// ---------------------------------------------------------------------------------------------
void Model::wgrad(Rank& R, int slot, int M, int N, int K, const void* A, int64_t lda, const void* B, int64_t ldb,
                  int accumulate) {
  if (fused_ == nullptr || slots_[slot].offset >= weights_end_) {
    gemm(R, M, N, K, A, lda, 1, B, ldb, 1, static_cast<int>(Epi::kStoreF32), G(R, slot), N, nullptr, 0, nullptr,
         nullptr, 0, accumulate);
    return;
  }
  {
    // A weight with too few output tiles to fill the GPU (the shards of tensor-parallel layers):
    // its gradient is split-K-reduced into G, checked, and the slot updated by the flat AdamW
    // kernel, gated like the fused epilogue (same arithmetic, the flag read on the device)
    GemmParams q;
    q.M = M;
    q.N = N;
    q.K = K;
    q.a_mn_major = 1;
    q.b_mn_major = 1;
    q.lda = lda;
    q.ldb = ldb;
    q.ldc = N;
    static const bool split_on = [] {
      const char* e = std::getenv("SW_WGRAD_SPLITK");
      return !(e != nullptr && e[0] == '0');
    }();
    if (split_on && gemm_split_k(q) > 1) {
      // the [M, N] gradient can span adjacent slots (the fused q|k|v or gate|up weights)
      const Slot& s = slots_[slot];
      const int64_t n = static_cast<int64_t>(M) * N;
      gemm(R, M, N, K, A, lda, 1, B, ldb, 1, static_cast<int>(Epi::kStoreF32), G(R, slot), N);
      k::nonfinite_check(G(R, slot), n, d_flag_, stream_);
      k::adamw(P(R, slot), R.m + s.offset, R.v + s.offset, G(R, slot), W(R, slot), n, fused_->lr, fused_->b1,
               fused_->b2, fused_->eps, fused_->wd, fused_->c1, fused_->c2, stream_, d_flag_);
      launches_ += 2;
      return;
    }
  }
  // optimizer in the epilogue: the gradient never leaves the accumulator
  GemmParams p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.A = A;
  p.lda = lda;
  p.a_mn_major = 1;
  p.B = B;
  p.ldb = ldb;
  p.b_mn_major = 1;
  p.epi = Epi::kAdamW;
  p.ldc = N;
  p.adam_p = P(R, slot);
  p.adam_m = R.m + slots_[slot].offset;
  p.adam_v = R.v + slots_[slot].offset;
  p.adam_w = W(R, slot);
  p.adam_flag = d_flag_;
  p.adam_lr = fused_->lr;
  p.adam_b1 = fused_->b1;
  p.adam_b2 = fused_->b2;
  p.adam_eps = fused_->eps;
  p.adam_wd = fused_->wd;
  p.adam_c1 = fused_->c1;
  p.adam_c2 = fused_->c2;
  tic();
  cuda_check(gemm_bf16(p, stream_), "gemm launch");
  toc(kProfGemm, 2.0 * M * N * static_cast<double>(K));
  if (prof_) {
    prof_tag_.resize(prof_rec_.size());
    prof_tag_.back() = "gemm," + std::to_string(M) + "," + std::to_string(N) + "," + std::to_string(K) + ",adamw,A_mn,B_mn";
  }
  ++launches_;
}

cudaEvent_t Model::on_side(const std::function<void()>& f) {
  if (side_ == nullptr || prof_) {  // profiling times every launch on stream_
    f();
    return nullptr;
  }
  // every wait on these events is enqueued within the same backward (it ends joined), so the
  // pool restarts at 0 each backward without re-recording an event that still has a wait due
  while (side_ev_.size() < side_next_ + 2) {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    side_ev_.push_back(e);
  }
  cudaEvent_t fork = side_ev_[side_next_++];
  cudaEvent_t done = side_ev_[side_next_++];
  cuda_check(cudaEventRecord(fork, stream_), "cudaEventRecord");
  cuda_check(cudaStreamWaitEvent(side_, fork, 0), "cudaStreamWaitEvent");
  // f() launches on stream_ (swapped with side_); the guard swaps them back even when f()
  // throws (a GEMM shape error, a launch failure) and then joins the side stream, so stream()
  // stays the model stream and no fork is left dangling
  struct Swap {
    Model* m;
    cudaEvent_t done;
    bool ok;
    ~Swap() {
      std::swap(m->stream_, m->side_);
      if (!ok && cudaEventRecord(done, m->side_) == cudaSuccess) cudaStreamWaitEvent(m->stream_, done, 0);
    }
  };
  {
    Swap guard{this, done, false};
    std::swap(stream_, side_);
    f();
    guard.ok = true;
  }
  cuda_check(cudaEventRecord(done, side_), "cudaEventRecord");
  return done;
}

void Model::main_wait(cudaEvent_t e) {
  if (e != nullptr) cuda_check(cudaStreamWaitEvent(stream_, e, 0), "cudaStreamWaitEvent");
}

void Model::backward_replica(std::vector<Rank*>& grp, bool accumulate) {
  const int64_t M = M_;
  const int d = d_, dl = dl_, fl = fl_;
  const int acc = accumulate ? 1 : 0;
  const bool tied = head_ < 0;
  const int head = tied ? tok_ : head_;
  // slots updated with atomics start from zero unless accumulating
  if (!accumulate) {
    for (Rank* R : grp) {
      auto zero = [&](int s) {
        if (s >= 0) cuda_check(cudaMemsetAsync(G(*R, s), 0, slots_[s].numel * 4, stream_), "memset");
      };
      for (const LayerSlots& ls : layers_) {
        zero(ls.ln1_s);
        zero(ls.ln1_b);
        zero(ls.ln2_s);
        zero(ls.ln2_b);
        zero(ls.o_b);    // o / fc2 bias gradients: column sums fused into the LayerNorm backward
        zero(ls.fc2_b);  // that consumes the same residual gradient (added per row chunk)
      }
      zero(lnf_s_);
      zero(lnf_b_);
      if (!tied) zero(tok_);
      if (T_ < S_) {
        cuda_check(cudaMemsetAsync(G(*R, pos_) + static_cast<int64_t>(T_) * d, 0,
                                   static_cast<int64_t>(S_ - T_) * d * 4, stream_),
                   "memset");
      }
    }
  }
  // Every weight's dgrad (which reads the bf16 shadow) is issued before its wgrad, so a wgrad
  // that applies AdamW in its epilogue never races a reader of the old weights.
  {
    // d(final_h) = dlogits . W_head (partial over the vocab shards when the head is split)
    auto prod = [&](Rank& R, int64_t r0, int64_t rows) {
      gemm(R, static_cast<int>(rows), d, vl_, R.logits + r0 * ldv_, ldv_, 0, W(R, head), d, 1,
           static_cast<int>(Epi::kStoreF32), R.dx + r0 * d, d);
    };
    auto cons = [&](Rank& R, int64_t r0, int64_t rows) {
      tic();
      k::layernorm_bwd(R.hs[L_] + r0 * d, R.statsf + r0, R.statsf + M + r0, P(R, lnf_s_), R.dx + r0 * d,
                       R.gres + r0 * d, R.gb + r0 * d, G(R, lnf_s_), Gn(R, lnf_b_), rows, d, 0, stream_, R.ln_partials,
                       spec_.rmsnorm, Gn(R, layers_[L_ - 1].fc2_b));
      toc(kProfNorm, 18.0 * rows * d);
      ++launches_;
    };
    if (th_ > 1) {
      row_ar(grp, &Rank::dx, [&](Rank& R) -> const bf16* { return R.logits; }, ldv_, vl_, head, 1,
             [&](Rank& R, int64_t r0, int64_t rows, const float* f32, const bf16* b16) {
               tic();
               if (b16 != nullptr)
                 k::layernorm_bwd(R.hs[L_] + r0 * d, R.statsf + r0, R.statsf + M + r0, P(R, lnf_s_), b16,
                                  R.gres + r0 * d, R.gb + r0 * d, G(R, lnf_s_), Gn(R, lnf_b_), rows, d, 0, stream_,
                                  R.ln_partials, spec_.rmsnorm, Gn(R, layers_[L_ - 1].fc2_b));
               else
                 k::layernorm_bwd(R.hs[L_] + r0 * d, R.statsf + r0, R.statsf + M + r0, P(R, lnf_s_), f32,
                                  R.gres + r0 * d, R.gb + r0 * d, G(R, lnf_s_), Gn(R, lnf_b_), rows, d, 0, stream_,
                                  R.ln_partials, spec_.rmsnorm, Gn(R, layers_[L_ - 1].fc2_b));
               toc(kProfNorm, 18.0 * rows * d);
               ++launches_;
             });
    } else {
      for (Rank* R : grp) prod(*R, 0, M);
      for (Rank* R : grp) cons(*R, 0, M);
    }
  }
  // side-stream events: a wgrad's inputs may be overwritten only after its event
  side_next_ = 0;
  cudaEvent_t ev_last = on_side([&] {
    for (Rank* R : grp) {
      // dW_head (+)= dlogits^T . final_h
      wgrad(*R, head, vl_, d, static_cast<int>(M), R->logits, ldv_, R->f, d, acc);
    }
  });
  cudaEvent_t ev_fc1 = nullptr, ev_qkv = nullptr;
  for (int l = L_ - 1; l >= 0; --l) {
    const LayerSlots& ls = layers_[l];
    main_wait(ev_fc1);  // the previous layer's fc1 wgrad has read dpre
    // ---- MLP ----
    // SwiGLU: dpre = d(gate) | d(up) [M, 2*fl] against the fused [gate; up] weight at gate_k
    const int fw = spec_.swiglu ? 2 * fl : fl;
    const int fk = spec_.swiglu ? ls.gate_k : ls.fc1_k;
    cudaEvent_t ev_fc2 = nullptr, ev_o = nullptr;
    for (Rank* R : grp) {
      bool cs_done = false;
      if (spec_.swiglu) {
        gemm(*R, static_cast<int>(M), fl, d, R->gb, d, 0, W(*R, ls.fc2_k), fl, 1,
             static_cast<int>(Epi::kSwiGLUBwd), R->dpre, 2 * fl, nullptr, 0, nullptr, R->pre[l], 2 * fl, 0, 0, 0,
             fl);
      } else {
        // the fc1 bias gradient's per-32-row column sums come out of the same epilogue
        GemmParams q;
        q.M = static_cast<int>(M);
        q.N = fl;
        q.K = d;
        q.b_mn_major = 1;
        q.epi = Epi::kGeluBwd;
        const bool fuse_cs = ls.fc1_b >= 0 && fuse_colsum_ && gemm_colsum_ok(q);
        gemm(*R, static_cast<int>(M), fl, d, R->gb, d, 0, W(*R, ls.fc2_k), fl, 1,
             static_cast<int>(Epi::kGeluBwd), R->dpre, fl, nullptr, 0, nullptr, R->pre[l], fl, 0, 0, 0, 0,
             nullptr, 0, fuse_cs ? R->col_scratch : nullptr);
        if (fuse_cs) {
          k::colsum_chunks(R->col_scratch, static_cast<int>((M + 31) / 32), fl, G(*R, ls.fc1_b) + R->mpi * fl, acc,
                           stream_);
          ++launches_;
          cs_done = true;
        }
      }
      ev_fc2 = on_side([&] { wgrad(*R, ls.fc2_k, d, fl, static_cast<int>(M), R->gb, d, R->act[l], fl, acc); });
      if (ls.fc1_b >= 0 && !cs_done) {
        k::colsum_bf16(R->dpre, fl, M, fl, 0, G(*R, ls.fc1_b) + R->mpi * fl, nullptr, nullptr, acc,
                       R->col_scratch, stream_);
        launches_ += 2;
      }
    }
    {
      auto prod = [&](Rank& R, int64_t r0, int64_t rows) {
        gemm(R, static_cast<int>(rows), d, fw, R.dpre + r0 * fw, fw, 0, W(R, fk), d, 1,
             static_cast<int>(Epi::kStoreF32), R.dx + r0 * d, d);
      };
      auto cons = [&](Rank& R, int64_t r0, int64_t rows) {
        main_wait(ev_fc2);  // the fc2 wgrad has read gb
        tic();
        k::layernorm_bwd(R.hmid[l] + r0 * d, R.stats2[l] + r0, R.stats2[l] + M + r0, P(R, ls.ln2_s), R.dx + r0 * d,
                         R.gres + r0 * d, R.gb + r0 * d, G(R, ls.ln2_s), Gn(R, ls.ln2_b), rows, d, 1, stream_,
                         R.ln_partials, spec_.rmsnorm, G(R, ls.o_b));
        toc(kProfNorm, 18.0 * rows * d);
        ++launches_;
      };
      if (tm_ > 1) {
        row_ar(grp, &Rank::dx, [&](Rank& R) -> const bf16* { return R.dpre; }, fw, fw, fk, 1,
               [&](Rank& R, int64_t r0, int64_t rows, const float* f32, const bf16* b16) {
                 main_wait(ev_fc2);
                 tic();
                 if (b16 != nullptr)
                   k::layernorm_bwd(R.hmid[l] + r0 * d, R.stats2[l] + r0, R.stats2[l] + M + r0, P(R, ls.ln2_s), b16,
                                    R.gres + r0 * d, R.gb + r0 * d, G(R, ls.ln2_s), Gn(R, ls.ln2_b), rows, d, 1,
                                    stream_, R.ln_partials, spec_.rmsnorm, G(R, ls.o_b));
                 else
                   k::layernorm_bwd(R.hmid[l] + r0 * d, R.stats2[l] + r0, R.stats2[l] + M + r0, P(R, ls.ln2_s), f32,
                                    R.gres + r0 * d, R.gb + r0 * d, G(R, ls.ln2_s), Gn(R, ls.ln2_b), rows, d, 1,
                                    stream_, R.ln_partials, spec_.rmsnorm, G(R, ls.o_b));
                 toc(kProfNorm, 18.0 * rows * d);
                 ++launches_;
               });
      } else {
        for (Rank* R : grp) prod(*R, 0, M);
        for (Rank* R : grp) cons(*R, 0, M);
      }
    }
    ev_fc1 = on_side([&] {
      for (Rank* R : grp) wgrad(*R, fk, fw, d, static_cast<int>(M), R->dpre, fw, R->a2[l], d, acc);
    });
    // ---- attention ----
    for (Rank* R : grp) {
      const bool delta_ready = gemm_dout(*R, l, W(*R, ls.o_k));
      ev_o = on_side([&] { wgrad(*R, ls.o_k, d, dl, static_cast<int>(M), R->gb, d, R->o[l], dl, acc); });
      main_wait(ev_qkv);  // the previous layer's QKV wgrad has read dqkv
      tic();
      bool cs_done = false;
      k::attention_bwd(R->qkv[l], R->o[l], R->lse[l], R->dout, R->dqkv, R->attn_scratch, B_, T_, hl_, hd_,
                       stream_, delta_ready, fuse_colsum_ ? R->col_scratch : nullptr, &cs_done);
      toc(kProfAttnBwd, 4.0 * B_ * hl_ * static_cast<double>(T_) * T_ * hd_);
      launches_ += delta_ready ? 2 : 3;
      if (cs_done) {  // the q|k|v bias gradients' partials came out of the attention backward
        k::colsum_chunks(R->col_scratch, static_cast<int>((M + 31) / 32), 3 * dl, G(*R, ls.q_b) + R->mpi * dl, acc,
                         stream_, dl, G(*R, ls.k_b) + R->mpi * dl, G(*R, ls.v_b) + R->mpi * dl);
        ++launches_;
      } else {
        k::colsum_bf16(R->dqkv, 3 * dl, M, 3 * dl, dl, G(*R, ls.q_b) + R->mpi * dl, G(*R, ls.k_b) + R->mpi * dl,
                       G(*R, ls.v_b) + R->mpi * dl, acc, R->col_scratch, stream_);
        launches_ += 2;
      }
    }
    {
      auto prod = [&](Rank& R, int64_t r0, int64_t rows) {
        gemm(R, static_cast<int>(rows), d, 3 * dl, R.dqkv + r0 * 3 * dl, 3 * dl, 0, W(R, ls.q_k), d, 1,
             static_cast<int>(Epi::kStoreF32), R.dx + r0 * d, d);
      };
      auto cons = [&](Rank& R, int64_t r0, int64_t rows) {
        main_wait(ev_o);  // the O-projection wgrad has read gb
        tic();
        k::layernorm_bwd(R.hs[l] + r0 * d, R.stats1[l] + r0, R.stats1[l] + M + r0, P(R, ls.ln1_s), R.dx + r0 * d,
                         R.gres + r0 * d, R.gb + r0 * d, G(R, ls.ln1_s), Gn(R, ls.ln1_b), rows, d, 1, stream_,
                         R.ln_partials, spec_.rmsnorm, (l > 0 ? Gn(R, layers_[l - 1].fc2_b) : nullptr));
        toc(kProfNorm, 18.0 * rows * d);
        ++launches_;
      };
      if (ta_ > 1) {
        row_ar(grp, &Rank::dx, [&](Rank& R) -> const bf16* { return R.dqkv; }, 3 * dl, 3 * dl, ls.q_k, 1,
               [&](Rank& R, int64_t r0, int64_t rows, const float* f32, const bf16* b16) {
                 main_wait(ev_o);
                 tic();
                 if (b16 != nullptr)
                   k::layernorm_bwd(R.hs[l] + r0 * d, R.stats1[l] + r0, R.stats1[l] + M + r0, P(R, ls.ln1_s), b16,
                                    R.gres + r0 * d, R.gb + r0 * d, G(R, ls.ln1_s), Gn(R, ls.ln1_b), rows, d, 1,
                                    stream_, R.ln_partials, spec_.rmsnorm, (l > 0 ? Gn(R, layers_[l - 1].fc2_b) : nullptr));
                 else
                   k::layernorm_bwd(R.hs[l] + r0 * d, R.stats1[l] + r0, R.stats1[l] + M + r0, P(R, ls.ln1_s), f32,
                                    R.gres + r0 * d, R.gb + r0 * d, G(R, ls.ln1_s), Gn(R, ls.ln1_b), rows, d, 1,
                                    stream_, R.ln_partials, spec_.rmsnorm, (l > 0 ? Gn(R, layers_[l - 1].fc2_b) : nullptr));
                 toc(kProfNorm, 18.0 * rows * d);
                 ++launches_;
               });
      } else {
        for (Rank* R : grp) prod(*R, 0, M);
        for (Rank* R : grp) cons(*R, 0, M);
      }
    }
    ev_qkv = on_side([&] {
      for (Rank* R : grp) wgrad(*R, ls.q_k, 3 * dl, d, static_cast<int>(M), R->dqkv, 3 * dl, R->a1[l], d, acc);
    });
    ev_last = ev_qkv;
    if (dp_overlap_) dp_bucket(grp, l, ev_qkv);
  }
  main_wait(ev_last);  // every wgrad (and its fused AdamW) done before anything downstream
  for (Rank* R : grp) {
    k::embed_bwd_pos(R->gres, G(*R, pos_), B_, T_, d, acc, stream_);
    k::embed_bwd_tok(R->tokens, R->gres, G(*R, tok_), M, d, spec_.vocab_size, R->tok_keys, stream_);
    launches_ += 2;
  }
  // column-parallel biases are replicated parameters: gather their gradient chunks
  // (the to_partition coercion of spmd.hpp:803-812).
  for (const LayerSlots& ls : layers_) {
    if (ta_ > 1) {
      ag_mp_slot(grp, ls.q_b, dl);
      ag_mp_slot(grp, ls.k_b, dl);
      ag_mp_slot(grp, ls.v_b, dl);
    }
    if (tm_ > 1 && ls.fc1_b >= 0) ag_mp_slot(grp, ls.fc1_b, fl);
  }
}

void Model::forward_backward(bool accumulate) {
  check_trainable("forward_backward");
  check_not_poisoned("forward_backward");
  cuda_check(cudaSetDevice(mesh_->cuda_device), "cudaSetDevice");
  launches_ = 0;
  if (dp_buckets_issued_) {  // a previous overlapped backward that never reached dp_sync
    cudaEvent_t e = dp_ev_[static_cast<size_t>(L_)];
    cuda_check(cudaEventRecord(e, dp_stream_), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(stream_, e, 0), "cudaStreamWaitEvent");
    dp_buckets_issued_ = false;
  }
  const int first = mesh_->emulated ? 0 : ranks_[0].dpi;
  const int last = mesh_->emulated ? mesh_->dp - 1 : ranks_[0].dpi;
  for (int r = first; r <= last; ++r) {
    std::vector<Rank*> grp = replica(r);
    forward_replica(grp, true);
    backward_replica(grp, accumulate);
  }
  cuda_check(cudaGetLastError(), "forward_backward");
}

void Model::forward_only() {
  cuda_check(cudaSetDevice(mesh_->cuda_device), "cudaSetDevice");
  const int first = mesh_->emulated ? 0 : ranks_[0].dpi;
  const int last = mesh_->emulated ? mesh_->dp - 1 : ranks_[0].dpi;
  for (int r = first; r <= last; ++r) {
    std::vector<Rank*> grp = replica(r);
    forward_replica(grp, false);
  }
  cuda_check(cudaGetLastError(), "forward");
}

void Model::scale_grads(double factor) {
  check_trainable("scale_grads");
  for (Rank& R : ranks_) {
    k::scale_f32(R.g, flat_n_, static_cast<float>(factor), stream_);
    ++launches_;
  }
}

void Model::dp_reduce_range(int64_t off, int64_t n, cudaStream_t s) {
  const float inv = 1.0f / static_cast<float>(mesh_->dp);
  for (int j = 0; j < mesh_->mp; ++j) {
    if (mesh_->emulated) {
      std::vector<float*> ptrs;
      for (int id : mesh_->dp_group(j)) ptrs.push_back(ranks_[id].g + off);
      k::sum_ranks_f32(ptrs.data(), static_cast<int>(ptrs.size()), n, inv, s);
      ++launches_;
    } else if (ranks_[0].mpi == j) {
      nccl_check(ncclAllReduce(ranks_[0].g + off, ranks_[0].g + off, n, ncclFloat, ncclSum, mesh_->dp_comm, s),
                 "AllReduce(dp)");
      k::scale_f32(ranks_[0].g + off, n, inv, s);
      ++launches_;
    }
  }
}

void Model::dp_bucket(std::vector<Rank*>& grp, int l, cudaEvent_t ready) {
  // emulated mesh: the replicas run one after another, so a layer's gradients are final once
  // the last replica's backward has produced them
  if (mesh_->emulated && grp[0]->dpi != mesh_->dp - 1) return;
  if (dp_stream_ == nullptr) {
    cuda_check(cudaStreamCreateWithFlags(&dp_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  }
  while (static_cast<int>(dp_ev_.size()) < L_ + 1) {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    dp_ev_.push_back(e);
  }
  if (ready == nullptr) {  // the wgrads ran on stream_
    ready = dp_ev_[static_cast<size_t>(l)];
    cuda_check(cudaEventRecord(ready, stream_), "cudaEventRecord");
  }
  cuda_check(cudaStreamWaitEvent(dp_stream_, ready, 0), "cudaStreamWaitEvent");
  const LayerSlots& ls = layers_[l];
  const int64_t off = slots_[ls.q_k].offset;
  const int64_t end = slots_[ls.fc2_k].offset + slots_[ls.fc2_k].numel;
  dp_reduce_range(off, end - off, dp_stream_);
  dp_buckets_issued_ = true;
}

void Model::dp_sync() {
  check_trainable("dp_sync_grads");
  if (mesh_->dp == 1) return;
  if (dp_buckets_issued_) {
    // the layers' GEMM-weight gradients were reduced during the backward: join, then the rest
    cudaEvent_t e = dp_ev_[static_cast<size_t>(L_)];
    cuda_check(cudaEventRecord(e, dp_stream_), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(stream_, e, 0), "cudaStreamWaitEvent");
    dp_reduce_range(layers_end_, flat_n_ - layers_end_, stream_);
    dp_buckets_issued_ = false;
  } else {
    dp_reduce_range(0, flat_n_, stream_);
  }
  for (int j = 0; j < mesh_->mp; ++j)
    mesh_->record(CollKind::kAllReduce, mesh_->dp_group(j), static_cast<uint64_t>(flat_n_) * 4);
}

void Model::adamw(double lr, double b1, double b2, double eps, double wd, bool check_finite) {
  check_trainable("adamw_step");
  check_not_poisoned("adamw_step");
  if (check_finite) {
    cuda_check(cudaMemsetAsync(d_flag_, 0, sizeof(int), stream_), "memset");
    for (Rank& R : ranks_) {
      k::nonfinite_check(R.g, flat_n_, d_flag_, stream_);
      ++launches_;
    }
    int flag = 0;
    cuda_check(cudaMemcpyAsync(&flag, d_flag_, sizeof(int), cudaMemcpyDeviceToHost, stream_), "D2H");
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    if (flag) {
      // slow path: name the first offending parameter like train_state.hpp:207-210
      std::vector<float> host;
      for (const Slot& s : slots_) {
        for (Rank& R : ranks_) {
          host.resize(s.numel);
          cuda_check(cudaMemcpy(host.data(), R.g + s.offset, s.numel * 4, cudaMemcpyDeviceToHost), "D2H");
          for (float x : host) {
            if (!std::isfinite(x)) {
              fail(SW_ERR_NONFINITE, "adamw_step: non-finite gradient for parameter '" + s.name + "'");
            }
          }
        }
      }
      fail(SW_ERR_NONFINITE, "adamw_step: non-finite gradient");
    }
  }
  const double t = static_cast<double>(step_ + 1);
  const float c1 = static_cast<float>(1.0 - std::pow(b1, t));
  const float c2 = static_cast<float>(1.0 - std::pow(b2, t));
  for (Rank& R : ranks_) {
    tic();
    k::adamw(R.p, R.m, R.v, R.g, R.w, flat_n_, static_cast<float>(lr), static_cast<float>(b1),
             static_cast<float>(b2), static_cast<float>(eps), static_cast<float>(wd), c1, c2, stream_);
    toc(kProfAdamw, 30.0 * flat_n_);
    ++launches_;
  }
  ++step_;
  cuda_check(cudaGetLastError(), "adamw");
}

void Model::fail_no_fp32_weight() {
  fail(SW_ERR_CONFIG, "inference-only model: GEMM weights are held in bf16 only");
}

void Model::check_trainable(const char* what) const {
  if (inference_) fail(SW_ERR_CONFIG, std::string(what) + ": this is an inference-only model (no gradients or optimizer state)");
}

void Model::check_not_poisoned(const char* what) const {
  if (poisoned_) {
    fail(SW_ERR_NONFINITE, std::string(what) + ": the model state was left half-updated by a non-finite fused "
                           "optimizer step; call init_params or load_checkpoint first");
  }
}

bool Model::train_step(double lr, double b1, double b2, double eps, double wd) {
  check_trainable("train_step");
  check_not_poisoned("train_step");
  static const bool disabled = [] {
    const char* e = std::getenv("SW_FUSED_ADAMW");
    return e != nullptr && e[0] == '0';
  }();
  if (disabled || mesh_->dp != 1) {
    static const bool overlap = [] {
      const char* e = std::getenv("SW_DP_OVERLAP");
      return !(e != nullptr && e[0] == '0');
    }();
    dp_overlap_ = overlap && mesh_->dp > 1;
    try {
      forward_backward(false);
    } catch (...) {
      dp_overlap_ = false;
      throw;
    }
    dp_overlap_ = false;
    dp_sync();
    adamw(lr, b1, b2, eps, wd, true);
    return false;
  }
  // Optimizer in the backward (dp == 1, no accumulation): every GEMM weight is updated by its
  // wgrad epilogue; the small parameters (embeddings, biases, LayerNorm) by one flat AdamW.
  const double t = static_cast<double>(step_ + 1);
  FusedAdam fa;
  fa.lr = static_cast<float>(lr);
  fa.b1 = static_cast<float>(b1);
  fa.b2 = static_cast<float>(b2);
  fa.eps = static_cast<float>(eps);
  fa.wd = static_cast<float>(wd);
  fa.c1 = static_cast<float>(1.0 - std::pow(b1, t));
  fa.c2 = static_cast<float>(1.0 - std::pow(b2, t));
  cuda_check(cudaMemsetAsync(d_flag_, 0, sizeof(int), stream_), "memset");
  fused_ = &fa;
  try {
    forward_backward(false);
  } catch (...) {
    fused_ = nullptr;
    throw;
  }
  fused_ = nullptr;
  const int64_t n_small = flat_n_ - weights_end_;
  for (Rank& R : ranks_) {
    k::nonfinite_check(R.g + weights_end_, n_small, d_flag_, stream_);
    ++launches_;
  }
  int flag = 0;
  cuda_check(cudaMemcpyAsync(&flag, d_flag_, sizeof(int), cudaMemcpyDeviceToHost, stream_), "D2H");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  if (flag & 2) {
    // The loss was non-finite, so every fused epilogue skipped its update (bit 2 was set before
    // the backward began): the state is exactly as before the step. Redo the step the
    // reference's way (check every gradient, then update) so the error names the parameter of
    // train_state.hpp:207-210, or the update goes ahead if the gradients are finite after all.
    forward_backward(false);
    adamw(lr, b1, b2, eps, wd, true);
    return false;
  }
  if (flag) {
    // finite loss, non-finite gradient found inside the backward: the wgrad epilogues that ran
    // before it was flagged already updated their GEMM weights, so the state is half-updated
    poisoned_ = true;
    fail(SW_ERR_NONFINITE, "adamw_step: non-finite gradient (optimizer fused into the backward: some GEMM "
                           "weights of this step were already updated; the model refuses further steps "
                           "and checkpoints until init_params or load_checkpoint)");
  }
  for (Rank& R : ranks_) {
    tic();
    k::adamw(R.p + weights_end_, R.m + weights_end_, R.v + weights_end_, R.g + weights_end_, R.w + weights_end_,
             n_small, fa.lr, fa.b1, fa.b2, fa.eps, fa.wd, fa.c1, fa.c2, stream_);
    toc(kProfAdamw, 30.0 * n_small);
    ++launches_;
  }
  ++step_;
  cuda_check(cudaGetLastError(), "train_step");
  return true;
}

// ---------------------------------------------------------------------------------------------
// greedy generation
// ---------------------------------------------------------------------------------------------
void Model::pick_tokens(std::vector<Rank*>& grp, const std::vector<const bf16*>& rows, int64_t stride) {
  const int B = B_;
  for (size_t i = 0; i < grp.size(); ++i) {
    Rank& R = *grp[i];
    DecodeBufs& D = dec_[static_cast<size_t>(&R - ranks_.data())];
    const int shard = th_ > 1 ? R.mpi : 0;
    if (th_ > 1) cuda_check(cudaMemsetAsync(D.arg, 0, sizeof(float) * 2 * B * th_, stream_), "memset");
    k::argmax_rows(rows[i], stride, B, vl_, shard * vl_, D.arg + static_cast<int64_t>(shard) * 2 * B, stream_,
                   D.argpart);
    launches_ += 2;
  }
  if (th_ > 1) {
    std::vector<float*> ptrs;
    for (Rank* R : grp) ptrs.push_back(dec_[static_cast<size_t>(R - ranks_.data())].arg);
    ar_mp_ptrs(grp, ptrs, static_cast<int64_t>(2) * B * th_);  // all-gather by summing disjoint slots
  }
  for (Rank* R : grp) {
    DecodeBufs& D = dec_[static_cast<size_t>(R - ranks_.data())];
    k::argmax_combine(D.arg, th_, B, D.tok, stream_);
    ++launches_;
  }
}

void Model::shift_rows(std::vector<Rank*>& grp, int64_t rows) {
  const int64_t d = d_, mp = mesh_->mp;
  auto mv = [rows](auto& ptr, int64_t per_row) {
    if (ptr != nullptr) ptr += rows * per_row;
  };
  for (Rank* R : grp) {
    for (int l = 0; l <= L_; ++l) mv(R->hs[l], d);
    for (int l = 0; l < L_; ++l) {
      mv(R->hmid[l], d);
      mv(R->stats1[l], 1);
      mv(R->stats2[l], 1);
      mv(R->a1[l], d);
      mv(R->a2[l], d);
      mv(R->qkv[l], 3 * dl_);
      mv(R->o[l], dl_);
      mv(R->lse[l], hl_);
      mv(R->pre[l], fl_ * (spec_.swiglu ? 2 : 1));
      mv(R->act[l], fl_);
    }
    mv(R->statsf, 1);
    mv(R->f, d);
    mv(R->logits, ldv_);
    mv(R->tokens, 1);
    mv(R->targets, 1);
    mv(R->weights, 1);
    mv(R->wloss, 1);
    mv(R->part, d);
    mv(R->arb, d);
    mv(R->xstats, 2 * mp);
    mv(R->xt, 1);
    mv(R->xlse, 1);
  }
}

void Model::window_forward(std::vector<Rank*>& grp, const std::vector<std::vector<int32_t>>& ctx, int take) {
  // the reference's window (cli.cpp:435-440): the last `take` context tokens at positions
  // 0..take-1, zeros after; the causal mask keeps the padding out of position take-1
  std::vector<int32_t> win(static_cast<size_t>(M_), 0);
  for (int b = 0; b < B_; ++b) {
    const std::vector<int32_t>& c = ctx[static_cast<size_t>(b)];
    for (int j = 0; j < take; ++j) win[static_cast<size_t>(b) * T_ + j] = c[c.size() - take + j];
  }
  for (Rank* R : grp) {
    cuda_check(cudaMemcpyAsync(R->tokens, win.data(), M_ * 4, cudaMemcpyHostToDevice, stream_), "H2D");
    cuda_check(cudaMemsetAsync(R->targets, 0, M_ * 4, stream_), "memset");
    k::fill_f32(R->weights, M_, 1.0f, stream_);
    ++launches_;
  }
  // Causality makes rows >= take irrelevant to the logits of row take-1 and to the K/V cache
  // rows a later cached step reads (< take; it writes row p itself before attending to it), so
  // a short prompt's prefill runs only the first Tp = take rounded up to 128 rows of each
  // sequence, one sequence at a time (SW_PREFILL_TRIM=0: the whole window, as the reference).
  static const bool trim_on = [] {
    const char* e = std::getenv("SW_PREFILL_TRIM");
    return !(e != nullptr && e[0] == '0');
  }();
  const int Tp = (take + 127) / 128 * 128;
  if (trim_on && Tp < T_ && B_ > 1 && T_ >= 2 * Tp) {
    // Several sequences: their first Tp rows side by side ([B, Tp] rows) in one forward (GEMMs
    // of B * Tp rows instead of B launches of Tp), then each sequence's K/V rows move to its
    // [B, T] cache rows. Sequence b's packed rows [b Tp, b Tp + Tp) lie below every later
    // sequence's destination and T >= 2 Tp keeps a destination off its own source, so moving
    // b = B-1 down to 1 never overwrites a row that is still to be read.
    const int B = B_, T = T_, chunks = ar_chunks_;
    const int64_t M = M_;
    std::vector<int32_t> packed(static_cast<size_t>(B) * Tp, 0);
    for (int b = 0; b < B; ++b)
      std::copy(win.begin() + static_cast<int64_t>(b) * T, win.begin() + static_cast<int64_t>(b) * T + Tp,
                packed.begin() + static_cast<int64_t>(b) * Tp);
    for (Rank* R : grp) {
      cuda_check(cudaMemcpyAsync(R->tokens, packed.data(), packed.size() * 4, cudaMemcpyHostToDevice, stream_),
                 "H2D");
    }
    cuda_check(cudaStreamSynchronize(stream_), "prefill");  // `packed` is a host temporary
    T_ = Tp;
    M_ = static_cast<int64_t>(B) * Tp;
    if (M_ % ar_chunks_ != 0) ar_chunks_ = 1;
    head_row_ = take - 1;
    try {
      forward_replica(grp, false);
    } catch (...) {
      T_ = T;
      M_ = M;
      ar_chunks_ = chunks;
      head_row_ = -1;
      throw;
    }
    T_ = T;
    M_ = M;
    ar_chunks_ = chunks;
    head_row_ = -1;
    const int64_t row = 3LL * dl_;
    for (Rank* R : grp) {
      for (int l = 0; l < L_; ++l) {
        for (int b = B - 1; b >= 1; --b) {
          cuda_check(cudaMemcpyAsync(R->qkv[l] + static_cast<int64_t>(b) * T * row,
                                     R->qkv[l] + static_cast<int64_t>(b) * Tp * row, static_cast<size_t>(Tp) * row * 2,
                                     cudaMemcpyDeviceToDevice, stream_),
                     "D2D");
        }
      }
    }
    std::vector<const bf16*> rows;
    for (Rank* R : grp) rows.push_back(dec_[static_cast<size_t>(R - ranks_.data())].logits);
    pick_tokens(grp, rows, ldv_);
    return;
  }
  if (trim_on && Tp < T_) {
    const int B = B_, T = T_, chunks = ar_chunks_;
    const int64_t M = M_;
    B_ = 1;
    T_ = Tp;
    M_ = Tp;
    if (Tp % ar_chunks_ != 0) ar_chunks_ = 1;
    int shifted = 0;
    auto restore = [&] {
      shift_rows(grp, -static_cast<int64_t>(shifted) * T);
      B_ = B;
      T_ = T;
      M_ = M;
      ar_chunks_ = chunks;
    };
    head_row_ = take - 1;
    try {
      for (int b = 0; b < B; ++b) {
        head_seq_ = b;
        forward_replica(grp, false);
        if (b + 1 < B) {
          shift_rows(grp, T);
          ++shifted;
        }
      }
    } catch (...) {
      restore();
      head_row_ = -1;
      head_seq_ = 0;
      throw;
    }
    restore();
    head_row_ = -1;
    head_seq_ = 0;
  } else {
    head_row_ = take - 1;
    try {
      forward_replica(grp, false);
    } catch (...) {
      head_row_ = -1;
      throw;
    }
    head_row_ = -1;
  }
  std::vector<const bf16*> rows;
  for (Rank* R : grp) rows.push_back(dec_[static_cast<size_t>(R - ranks_.data())].logits);
  pick_tokens(grp, rows, ldv_);
}

void Model::decode_step(std::vector<Rank*>& grp, int p) {
  const int B = B_, d = d_, dl = dl_, fl = fl_;
  static const int pdl_on = [] {
    const char* e = std::getenv("SW_DECODE_PDL");
    return e != nullptr ? std::atoi(e) : 3;
  }();
  struct PdlScope {
    int& f;
    PdlScope(int& flag, int v) : f(flag) { f = v; }
    ~PdlScope() { f = 0; }
  } pdl_scope(pdl_, pdl_on);
  const bool dev_pos = p < 0;
  auto pd = [&](Rank& R) -> const int* { return dev_pos ? dec_[static_cast<size_t>(&R - ranks_.data())].pos : nullptr; };
  for (Rank* R : grp) {
    DecodeBufs& D = dec_[static_cast<size_t>(R - ranks_.data())];
    k::embed_rows(D.tok, P(*R, tok_), P(*R, pos_), p, D.x, B, d, stream_, pd(*R));
    ++launches_;
  }
  auto each = [&](auto&& fn) {
    for (Rank* R : grp) fn(*R, dec_[static_cast<size_t>(R - ranks_.data())]);
  };
  auto reduce = [&](float* DecodeBufs::*buf, int64_t n) {
    std::vector<float*> ptrs;
    for (Rank* R : grp) ptrs.push_back(dec_[static_cast<size_t>(R - ranks_.data())].*buf);
    ar_mp_ptrs(grp, ptrs, n);
  };
  for (int l = 0; l < L_; ++l) {
    const LayerSlots& ls = layers_[l];
    each([&](Rank& R, DecodeBufs& D) {
      k::layernorm_fwd_small(D.x, P(R, ls.ln1_s), Pn(R, ls.ln1_b), D.a, D.stats, D.stats + B, B, d, 1e-5f, stream_,
                       spec_.rmsnorm);
      ++launches_;
      gemm(R, B, 3 * dl, d, D.a, d, 0, W(R, ls.q_k), d, 0, static_cast<int>(Epi::kStoreBf16), D.qkv, 3 * dl, nullptr,
           0, P(R, ls.q_b) + R.mpi * dl, nullptr, 0, 0, dl, d);
      if (k::decode_attention_split(D.qkv, R.qkv[l], D.o, B, T_, p, hl_, hd_, stream_, pd(R), D.attn_part,
                                    D.attn_ticket)) {
        ++launches_;
      } else {
        k::kv_scatter(D.qkv, R.qkv[l], B, T_, p, dl, stream_, pd(R));
        k::decode_attention(D.qkv, R.qkv[l], D.o, B, T_, p, hl_, hd_, stream_, pd(R));
        launches_ += 2;
      }
      if (ta_ == 1) {
        gemm(R, B, d, dl, D.o, dl, 0, W(R, ls.o_k), dl, 0, static_cast<int>(Epi::kResidF32), D.xmid, d, nullptr, 0,
             P(R, ls.o_b), D.x, d);
      } else {
        gemm(R, B, d, dl, D.o, dl, 0, W(R, ls.o_k), dl, 0, static_cast<int>(Epi::kStoreF32), D.part, d);
      }
    });
    if (ta_ > 1) {
      reduce(&DecodeBufs::part, static_cast<int64_t>(B) * d);
      each([&](Rank& R, DecodeBufs& D) {
        k::add_residual_bias(D.x, D.part, P(R, ls.o_b), D.xmid, B, d, stream_);
        ++launches_;
      });
    }
    each([&](Rank& R, DecodeBufs& D) {
      k::layernorm_fwd_small(D.xmid, P(R, ls.ln2_s), Pn(R, ls.ln2_b), D.a, D.stats, D.stats + B, B, d, 1e-5f, stream_,
                       spec_.rmsnorm);
      ++launches_;
      if (spec_.swiglu) {
        gemm(R, B, fl, d, D.a, d, 0, W(R, ls.gate_k), d, 0, static_cast<int>(Epi::kSwiGLU), D.h, fl, D.pre, 2 * fl,
             nullptr, nullptr, 0, 0, 0, 0, fl);
      } else {
        gemm(R, B, fl, d, D.a, d, 0, W(R, ls.fc1_k), d, 0, static_cast<int>(Epi::kBiasGelu), D.pre, fl, D.h, fl,
             P(R, ls.fc1_b) + R.mpi * fl);
      }
      if (tm_ == 1) {
        gemm(R, B, d, fl, D.h, fl, 0, W(R, ls.fc2_k), fl, 0, static_cast<int>(Epi::kResidF32), D.x, d, nullptr, 0,
             Pn(R, ls.fc2_b), D.xmid, d);
      } else {
        gemm(R, B, d, fl, D.h, fl, 0, W(R, ls.fc2_k), fl, 0, static_cast<int>(Epi::kStoreF32), D.part, d);
      }
    });
    if (tm_ > 1) {
      reduce(&DecodeBufs::part, static_cast<int64_t>(B) * d);
      each([&](Rank& R, DecodeBufs& D) {
        k::add_residual_bias(D.xmid, D.part, Pn(R, ls.fc2_b), D.x, B, d, stream_);
        ++launches_;
      });
    }
  }
  const int head = head_ >= 0 ? head_ : tok_;
  std::vector<const bf16*> rows;
  each([&](Rank& R, DecodeBufs& D) {
    k::layernorm_fwd_small(D.x, P(R, lnf_s_), Pn(R, lnf_b_), D.f, D.stats, D.stats + B, B, d, 1e-5f, stream_,
                     spec_.rmsnorm);
    ++launches_;
    gemm(R, B, vl_, d, D.f, d, 0, W(R, head), d, 0, static_cast<int>(Epi::kStoreBf16), D.logits, ldv_);
    rows.push_back(D.logits);
  });
  pick_tokens(grp, rows, ldv_);
  if (dev_pos) {
    each([&](Rank&, DecodeBufs& D) {
      k::bump_i32(D.pos, stream_);
      ++launches_;
    });
  }
}

void Model::generate(const int32_t* prompts, int P, int n_new, int32_t* out) {
  if (P < 1 || P > T_) {
    fail(SW_ERR_SHAPE, "generate: prompt length " + std::to_string(P) + " must be in [1, seq_len " +
                           std::to_string(T_) + "]");
  }
  if (n_new < 1) fail(SW_ERR_CONFIG, "generate: n_new must be positive");
  cuda_check(cudaSetDevice(mesh_->cuda_device), "cudaSetDevice");
  if (dec_.empty()) {
    const int64_t B = B_;
    for (size_t i = 0; i < ranks_.size(); ++i) {
      DecodeBufs D;
      D.x = alloc<float>(B * d_);
      D.xmid = alloc<float>(B * d_);
      D.part = alloc<float>(B * d_);
      D.stats = alloc<float>(2 * B);
      D.arg = alloc<float>(2 * B * th_);
      D.a = alloc<bf16>(B * d_);
      D.qkv = alloc<bf16>(B * 3 * dl_);
      D.o = alloc<bf16>(B * dl_);
      D.pre = alloc<bf16>(B * 2 * fl_);
      D.h = alloc<bf16>(B * fl_);
      D.f = alloc<bf16>(B * d_);
      D.logits = alloc<bf16>(B * ldv_);
      D.tok = alloc<int32_t>(B);
      D.pos = alloc<int>(1);
      D.attn_part = alloc<float>(B * hl_ * k::decode_split_count() * (hd_ + 2));
      D.attn_ticket = alloc<unsigned int>(B * hl_);
      D.argpart = alloc<float>(B * k::kArgmaxChunks * 2);
      cuda_check(cudaMemset(D.attn_ticket, 0, sizeof(unsigned int) * B * hl_), "memset");
      dec_.push_back(D);
    }
  }
  std::vector<Rank*> grp = replica(mesh_->emulated ? 0 : ranks_[0].dpi);
  DecodeBufs& D0 = dec_[static_cast<size_t>(grp[0] - ranks_.data())];
  std::vector<std::vector<int32_t>> ctx(static_cast<size_t>(B_));
  for (int b = 0; b < B_; ++b) ctx[static_cast<size_t>(b)].assign(prompts + static_cast<int64_t>(b) * P, prompts + static_cast<int64_t>(b + 1) * P);
  // Cached steps are data-independent of the host (the new token stays on the device, the
  // position is known), so they run back to back: each one is a single CUDA-graph launch (the
  // emulated mesh; NCCL ranks launch eagerly) whose tokens are copied into dec_out_ and read back
  // once, before the window slides or at the end. SW_DECODE_GRAPH=0: eager launches.
  static const bool graph_on = [] {
    const char* e = std::getenv("SW_DECODE_GRAPH");
    return !(e != nullptr && e[0] == '0');
  }();
  const bool use_graph = graph_on && mesh_->emulated && !prof_;
  if (dec_out_cap_ < static_cast<int64_t>(n_new) * B_) {
    if (dec_out_ != nullptr) cudaFree(dec_out_);
    dec_out_ = nullptr;
    cuda_check(cudaMalloc(&dec_out_, sizeof(int32_t) * n_new * B_), "cudaMalloc");
    dec_out_cap_ = static_cast<int64_t>(n_new) * B_;
  }
  std::vector<int32_t> tok(static_cast<size_t>(B_));
  int pending = 0;  // cached steps whose tokens are still only on the device
  auto flush = [&](int upto) {  // read back steps [upto - pending, upto)
    if (pending == 0) return;
    std::vector<int32_t> buf(static_cast<size_t>(pending) * B_);
    cuda_check(cudaMemcpyAsync(buf.data(), dec_out_, buf.size() * 4, cudaMemcpyDeviceToHost, stream_), "D2H");
    cuda_check(cudaStreamSynchronize(stream_), "generate");
    for (int j = 0; j < pending; ++j) {
      const int i = upto - pending + j;
      for (int b = 0; b < B_; ++b) {
        const int32_t t = buf[static_cast<size_t>(j) * B_ + b];
        out[static_cast<int64_t>(b) * n_new + i] = t;
        ctx[static_cast<size_t>(b)].push_back(t);
      }
    }
    pending = 0;
  };
  int len = P;  // context length before step i's token
  for (int i = 0; i < n_new; ++i, ++len) {
    if (i == 0 || len > T_) {
      flush(i);
      window_forward(grp, ctx, len < T_ ? len : T_);  // prefill, or the sliding window
      cuda_check(cudaMemcpyAsync(tok.data(), D0.tok, B_ * 4, cudaMemcpyDeviceToHost, stream_), "D2H");
      cuda_check(cudaStreamSynchronize(stream_), "generate");
      for (int b = 0; b < B_; ++b) {
        out[static_cast<int64_t>(b) * n_new + i] = tok[static_cast<size_t>(b)];
        ctx[static_cast<size_t>(b)].push_back(tok[static_cast<size_t>(b)]);
      }
      continue;
    }
    // the newest token sits at position len - 1
    if (pending == 0) {
      for (Rank* R : grp) {
        const int p0 = len - 1;
        cuda_check(cudaMemcpyAsync(dec_[static_cast<size_t>(R - ranks_.data())].pos, &p0, sizeof(int),
                                   cudaMemcpyHostToDevice, stream_),
                   "H2D");
        cuda_check(cudaStreamSynchronize(stream_), "generate");  // p0 is a stack value
      }
    }
    if (use_graph) {
      if (dec_graph_ == nullptr) {
        cudaGraph_t g = nullptr;
        cuda_check(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "capture");
        try {
          decode_step(grp, -1);
        } catch (...) {
          cudaStreamEndCapture(stream_, &g);
          if (g != nullptr) cudaGraphDestroy(g);
          throw;
        }
        cuda_check(cudaStreamEndCapture(stream_, &g), "capture");
        cuda_check(cudaGraphInstantiate(&dec_graph_, g, 0), "cudaGraphInstantiate");
        cudaGraphDestroy(g);
      }
      cuda_check(cudaGraphLaunch(dec_graph_, stream_), "cudaGraphLaunch");
    } else {
      decode_step(grp, -1);
    }
    cuda_check(cudaMemcpyAsync(dec_out_ + static_cast<int64_t>(pending) * B_, D0.tok, B_ * 4, cudaMemcpyDeviceToDevice,
                               stream_),
               "D2D");
    ++pending;
  }
  flush(n_new);
}

double Model::last_loss() {
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  double sum = 0.0;
  int n = 0;
  for (Rank& R : ranks_) {
    if (R.mpi != 0) continue;
    double x = 0.0;
    cuda_check(cudaMemcpy(&x, R.loss, sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    sum += x;
    ++n;
  }
  if (!mesh_->emulated && mesh_->dp > 1) {
    // mean over replicas: every rank contributes its replica's loss once per mp column
    double* tmp = nullptr;
    cuda_check(cudaMalloc(&tmp, sizeof(double)), "cudaMalloc");
    double x = 0.0;
    cuda_check(cudaMemcpy(&x, ranks_[0].loss, sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    cuda_check(cudaMemcpy(tmp, &x, sizeof(double), cudaMemcpyHostToDevice), "H2D");
    nccl_check(ncclAllReduce(tmp, tmp, 1, ncclDouble, ncclSum, mesh_->dp_comm, stream_), "AllReduce(loss)");
    cuda_check(cudaMemcpyAsync(&x, tmp, sizeof(double), cudaMemcpyDeviceToHost, stream_), "D2H");
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    cudaFree(tmp);
    return x / mesh_->dp;
  }
  return n > 0 ? sum / n : 0.0;
}

void Model::logits_to_host(float* out) {
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  std::vector<bf16> tmp(static_cast<size_t>(M_ * ldv_));
  const int first = mesh_->emulated ? 0 : ranks_[0].dpi;
  const int last = mesh_->emulated ? mesh_->dp - 1 : ranks_[0].dpi;
  for (int r = first; r <= last; ++r) {
    float* o = out + (mesh_->emulated ? static_cast<int64_t>(r) * M_ * V_ : 0);
    for (Rank* R : replica(r)) {
      if (th_ == 1 && R->mpi != 0) continue;
      cuda_check(cudaMemcpy(tmp.data(), R->logits, tmp.size() * 2, cudaMemcpyDeviceToHost), "D2H");
      const int64_t c0 = th_ == 1 ? 0 : static_cast<int64_t>(R->mpi) * vl_;
      for (int64_t i = 0; i < M_; ++i)
        for (int j = 0; j < vl_; ++j) o[i * V_ + c0 + j] = __bfloat162float(tmp[i * ldv_ + j]);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// profiling
// ---------------------------------------------------------------------------------------------
void Model::set_profiling(bool on) {
  prof_ = on;
  ev_next_ = 0;
  prof_rec_.clear();
  prof_tag_.clear();
}

void Model::tic(cudaStream_t s) {
  if (!prof_) return;
  if (s == nullptr) s = stream_;
  if (ev_next_ + 2 > events_.size()) {
    for (int i = 0; i < 256; ++i) {
      cudaEvent_t e;
      cuda_check(cudaEventCreate(&e), "cudaEventCreate");
      events_.push_back(e);
    }
  }
  cuda_check(cudaEventRecord(events_[ev_next_], s), "cudaEventRecord");
}

void Model::toc(int cat, double work, cudaStream_t s) {
  if (!prof_) return;
  if (s == nullptr) s = stream_;
  cuda_check(cudaEventRecord(events_[ev_next_ + 1], s), "cudaEventRecord");
  ev_next_ += 2;
  prof_rec_.emplace_back(cat, work);
}

void Model::read_profile(double* ms, double* work, int64_t* count) {
  for (int c = 0; c < kProfCats; ++c) {
    ms[c] = 0.0;
    work[c] = 0.0;
    count[c] = 0;
  }
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  cuda_check(cudaStreamSynchronize(comm_stream_), "sync");
  // SW_PROFILE_LOG=<path>: append one CSV line per timed launch (category, ms, work, tag)
  const char* log_path = std::getenv("SW_PROFILE_LOG");
  FILE* log = log_path != nullptr ? std::fopen(log_path, "a") : nullptr;
  prof_tag_.resize(prof_rec_.size());
  for (size_t i = 0; i < prof_rec_.size(); ++i) {
    float t = 0.f;
    cuda_check(cudaEventElapsedTime(&t, events_[2 * i], events_[2 * i + 1]), "cudaEventElapsedTime");
    const int c = prof_rec_[i].first;
    ms[c] += t;
    work[c] += prof_rec_[i].second;
    count[c] += 1;
    if (log != nullptr) std::fprintf(log, "%d,%.6f,%.6g,%s\n", c, t, prof_rec_[i].second, prof_tag_[i].c_str());
  }
  if (log != nullptr) std::fclose(log);
  ev_next_ = 0;
  prof_rec_.clear();
  prof_tag_.clear();
}

}  // namespace sw
