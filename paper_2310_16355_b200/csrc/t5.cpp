// GPU executor of the T5 encoder-decoder extension (see t5.h; oracle/t5_ref.py is the math).
#include "t5.h"

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "gemm.h"
#include "kernels.h"
#include "status.h"

namespace sw {

namespace {

uint64_t t5_mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

uint64_t t5_fnv1a(const std::string& s) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 0x100000001b3ull;
  }
  return h;
}

int64_t t5_numel(const Dims& d) {
  int64_t n = 1;
  for (int64_t x : d) n *= x;
  return n;
}

constexpr int64_t kT5Align = 64;
constexpr float kT5Eps = 1e-6f;  // T5LayerNorm

}  // namespace

T5Model::T5Model(const ModelSpec& spec, const Plan& plan, Mesh* mesh, int batch, int enc_len, int dec_len)
    : spec_(spec), plan_(plan), mesh_(mesh), B_(batch), Te_(enc_len), Td_(dec_len) {
  if (mesh == nullptr) fail(SW_ERR_CONFIG, "sw_t5_create: mesh is NULL");
  if (!spec.t5) fail(SW_ERR_CONFIG, "sw_t5_create: the model spec is not arch = t5");
  if (batch < 1 || enc_len < 1 || dec_len < 1) fail(SW_ERR_CONFIG, "sw_t5_create: sizes must be positive");
  if (enc_len > spec.max_seq_len || dec_len > spec.max_seq_len) {
    fail(SW_ERR_CONFIG, "sw_t5_create: sequence length exceeds max_seq_len " + std::to_string(spec.max_seq_len));
  }
  if (mesh->dp != 1) fail(SW_ERR_CONFIG, "sw_t5_create: the T5 executor runs dp = 1 (tensor parallel only)");
  if (plan.n_shards != mesh->mp) {
    fail(SW_ERR_CONFIG, "sw_t5_create: plan derived for " + std::to_string(plan.n_shards) +
                            " shards but the mesh has mp=" + std::to_string(mesh->mp));
  }
  Me_ = static_cast<int64_t>(B_) * Te_;
  Md_ = static_cast<int64_t>(B_) * Td_;
  Le_ = spec.n_layers;
  Ld_ = spec.n_dec_layers;
  d_ = static_cast<int>(spec.d_model);
  H_ = spec.n_heads;
  dk_ = static_cast<int>(spec.d_kv);
  inner_ = H_ * dk_;
  dff_ = static_cast<int>(spec.d_ff);
  V_ = static_cast<int>(spec.vocab_size);
  nb_ = spec.rel_buckets;
  maxd_ = spec.rel_max_distance;
  if (dk_ > 256) fail(SW_ERR_CONFIG, "sw_t5_create: d_kv > 256 is not supported by the attention kernels");
  fused_x_ = Te_ == Td_;
  {
    const char* e = std::getenv("SW_T5_TC");
    // tcgen05 attention for d_kv = 128: self-attention over the fused q|k|v rows (relative bias
    // as a LUT of 2T + 128 entries per head), cross-attention over separate q and encoder k|v
    tc_ = dk_ == 128 && (Te_ > Td_ ? Te_ : Td_) + 128 <= 4096 && !(e != nullptr && e[0] == '0');
  }
  cuda_check(cudaSetDevice(mesh->cuda_device), "cudaSetDevice");
  cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  build_layout();
  allocate();
}

T5Model::~T5Model() {
  if (stream_) cudaStreamSynchronize(stream_);
  for (cudaEvent_t e : events_) cudaEventDestroy(e);
  for (void* p : allocations_) cudaFree(p);
  if (stream_) cudaStreamDestroy(stream_);
}

template <typename T>
T* T5Model::alloc(int64_t n) {
  void* p = nullptr;
  const size_t bytes = static_cast<size_t>(n > 0 ? n : 1) * sizeof(T);
  cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
  allocations_.push_back(p);
  bytes_ += static_cast<int64_t>(bytes);
  return static_cast<T*>(p);
}

void T5Model::build_layout() {
  const int t = mesh_->mp;
  const std::vector<NamedShape> shapes = transformer_param_shapes(spec_);
  std::unordered_map<std::string, const NamedShape*> by_name;
  uint64_t draws = 0;
  std::unordered_map<std::string, uint64_t> draw_of;
  for (const auto& p : shapes) {
    by_name[p.name] = &p;
    const std::string leaf = p.name.substr(p.name.rfind('/') + 1);
    if (leaf != "scale" && leaf != "bias") {
      draw_of[p.name] = draws;
      draws += 2 * static_cast<uint64_t>(t5_numel(p.dims));
    }
  }
  int64_t off = 0;
  auto place = [&](const std::string& name, bool align) {
    const auto it = by_name.find(name);
    if (it == by_name.end()) fail(SW_ERR_CONFIG, "T5 layout: no parameter '" + name + "'");
    const NamedShape& p = *it->second;
    Slot s;
    s.name = name;
    s.global = p.dims;
    const Layout* l = plan_.find(name);
    if (l == nullptr) fail(SW_ERR_CONFIG, "ShardingPlan: no entry for parameter '" + name + "'");
    s.layout = *l;
    s.local = p.dims;
    if (l->kind == Layout::kSplit) {
      if (p.dims[l->dim] % t != 0) {
        fail(SW_ERR_PARTITION, "local_shape: dim " + std::to_string(l->dim) + " of " + dims_str(p.dims) +
                                   " is not divisible by " + std::to_string(t) + " shards");
      }
      s.local[l->dim] = p.dims[l->dim] / t;
    }
    s.numel = t5_numel(s.local);
    const std::string leaf = name.substr(name.rfind('/') + 1);
    s.init = leaf == "scale" ? 1 : 2;
    if (s.init == 2) {
      s.draw_base = draw_of[name];
      s.init_scale = name.rfind("embed/", 0) == 0 ? 0.02 : 1.0 / std::sqrt(static_cast<double>(p.dims[1]));
    }
    if (align) off = (off + kT5Align - 1) / kT5Align * kT5Align;
    s.offset = off;
    off += s.numel;
    slots_.push_back(s);
    slot_of_[name] = static_cast<int>(slots_.size()) - 1;
    return static_cast<int>(slots_.size()) - 1;
  };
  auto expect = [&](int s, Layout::Kind kind, int dim, const char* what) {
    const Layout& l = slots_[s].layout;
    const bool ok = l.kind == kind && (kind != Layout::kSplit || l.dim == dim);
    const bool rep = l.kind == Layout::kReplicated;
    if (!(ok || (t == 1 && rep))) {
      fail(SW_ERR_PARTITION, std::string("T5 executor: unsupported partition for ") + what + " '" +
                                 slots_[s].name + "' (supported: the reference rule layout)");
    }
  };
  // Region 1: the GEMM weight matrices (their wgrad epilogue can apply AdamW in place, see
  // train_step); region 2 from weights_end_: embedding, relative-position biases, norm scales.
  auto stack = [&](const std::string& st, int layers, bool decoder, std::vector<T5Layer>& out, bool gemm_pass) {
    out.resize(layers);
    for (int l = 0; l < layers; ++l) {
      const std::string b = st + "/block_" + std::to_string(l) + "/";
      T5Layer& L = out[l];
      if (!gemm_pass) {
        L.ln1 = place(b + "ln1/scale", true);
        if (l == 0) {
          const int rb = place(b + "attn/rel_bias/kernel", true);
          expect(rb, Layout::kReplicated, 0, "the relative-position bias");
          (decoder ? rb_d_ : rb_e_) = rb;
        }
        if (decoder) L.lnx = place(b + "ln_x/scale", true);
        L.ln2 = place(b + "ln2/scale", true);
        continue;
      }
      L.q = place(b + "attn/q/kernel", true);  // q|k|v adjacent: fused [3*inner/t, d]
      place(b + "attn/k/kernel", false);
      place(b + "attn/v/kernel", false);
      L.o = place(b + "attn/o/kernel", true);
      for (int s : {L.q, L.q + 1, L.q + 2}) expect(s, Layout::kSplit, 0, "attention q/k/v");
      expect(L.o, Layout::kSplit, 1, "attention o");
      if (decoder) {
        L.cq = place(b + "cross_attn/q/kernel", true);
        L.ck = place(b + "cross_attn/k/kernel", true);  // k|v adjacent: fused [2*inner/t, d]
        place(b + "cross_attn/v/kernel", false);
        L.co = place(b + "cross_attn/o/kernel", true);
        for (int s : {L.cq, L.ck, L.ck + 1}) expect(s, Layout::kSplit, 0, "cross-attention q/k/v");
        expect(L.co, Layout::kSplit, 1, "cross-attention o");
      }
      L.fc1 = place(b + "mlp/fc1/kernel", true);
      L.fc2 = place(b + "mlp/fc2/kernel", true);
      expect(L.fc1, Layout::kSplit, 0, "mlp fc1");
      expect(L.fc2, Layout::kSplit, 1, "mlp fc2");
    }
    if (!gemm_pass) (decoder ? lnf_d_ : lnf_e_) = place(st + "/final_ln/scale", true);
  };
  stack("enc", Le_, false, enc_, true);
  stack("dec", Ld_, true, dec_, true);
  head_ = place("lm_head/kernel", true);
  if (slots_[head_].layout.kind != Layout::kReplicated) {
    fail(SW_ERR_PARTITION, "T5 executor: lm_head/kernel must be replicated (the reference plan)");
  }
  weights_end_ = (off + kT5Align - 1) / kT5Align * kT5Align;
  off = weights_end_;
  tok_ = place("embed/tok/kernel", true);
  expect(tok_, Layout::kReplicated, 0, "the embedding");
  stack("enc", Le_, false, enc_, false);
  stack("dec", Ld_, true, dec_, false);
  for (const Slot& s : slots_) {
    if (s.global.size() < 2 && s.layout.kind != Layout::kReplicated) {
      fail(SW_ERR_PARTITION, "T5 executor: 1-D parameter '" + s.name + "' must be replicated");
    }
  }
  flat_n_ = (off + kT5Align - 1) / kT5Align * kT5Align;
  t_ = slots_[enc_[0].q].layout.kind == Layout::kSplit ? t : 1;
  if (H_ % t_ != 0) fail(SW_ERR_PARTITION, "T5 executor: n_heads not divisible by the attention split");
  hl_ = H_ / t_;
  il_ = inner_ / t_;
  fl_ = dff_ / t_;
  for (auto [what, v] : {std::pair<const char*, int>{"d_model", d_}, {"n_heads*d_kv/t", il_}, {"d_ff/t", fl_},
                         {"vocab", V_}}) {
    if (v % 8 != 0) {
      fail(SW_ERR_CONFIG, std::string("T5 executor: ") + what + " = " + std::to_string(v) +
                              " must be a multiple of 8 (16-byte TMA rows)");
    }
  }
}

void T5Model::allocate() {
  const int64_t Me = Me_, Md = Md_, Mx = Me > Md ? Me : Md;
  ld_cq_ = fused_x_ ? 3LL * il_ : il_;
  ld_ckv_ = fused_x_ ? 3LL * il_ : 2LL * il_;
  std::vector<int32_t> ids_e(static_cast<size_t>(Te_) * Te_), ids_d(static_cast<size_t>(Td_) * Td_);
  for (int i = 0; i < Te_; ++i)
    for (int j = 0; j < Te_; ++j) ids_e[static_cast<size_t>(i) * Te_ + j] = t5_rel_bucket(j - i, true, nb_, maxd_);
  for (int i = 0; i < Td_; ++i)
    for (int j = 0; j < Td_; ++j) ids_d[static_cast<size_t>(i) * Td_ + j] = t5_rel_bucket(j - i, false, nb_, maxd_);
  for (int dev : mesh_->local_devices()) {
    T5Rank R;
    R.device = dev;
    R.mpi = mesh_->mp_index(dev);
    R.p = alloc<float>(flat_n_);
    R.g = alloc<float>(flat_n_);
    R.m = alloc<float>(flat_n_);
    R.v = alloc<float>(flat_n_);
    R.w = alloc<bf16>(flat_n_);
    for (float* x : {R.p, R.g, R.m, R.v}) cuda_check(cudaMemsetAsync(x, 0, flat_n_ * 4, stream_), "memset");
    cuda_check(cudaMemsetAsync(R.w, 0, flat_n_ * 2, stream_), "memset");
    for (int l = 0; l <= Le_; ++l) R.hs_e.push_back(alloc<float>(Me * d_));
    for (int l = 0; l < Le_; ++l) {
      R.hm_e.push_back(alloc<float>(Me * d_));
      R.st1_e.push_back(alloc<float>(Me));
      R.st2_e.push_back(alloc<float>(Me));
      R.a1_e.push_back(alloc<bf16>(Me * d_));
      R.qkv_e.push_back(alloc<bf16>(Me * 3 * il_));
      R.o_e.push_back(alloc<bf16>(Me * il_));
      R.lse_e.push_back(alloc<float>(Me * hl_));
      R.a2_e.push_back(alloc<bf16>(Me * d_));
      R.act_e.push_back(alloc<bf16>(Me * fl_));
    }
    R.stf_e = alloc<float>(Me);
    R.eo = alloc<bf16>(Me * d_);
    for (int l = 0; l <= Ld_; ++l) R.hs_d.push_back(alloc<float>(Md * d_));
    for (int l = 0; l < Ld_; ++l) {
      R.hm_d.push_back(alloc<float>(Md * d_));
      R.hx_d.push_back(alloc<float>(Md * d_));
      R.st1_d.push_back(alloc<float>(Md));
      R.stx_d.push_back(alloc<float>(Md));
      R.st2_d.push_back(alloc<float>(Md));
      R.a1_d.push_back(alloc<bf16>(Md * d_));
      R.qkv_d.push_back(alloc<bf16>(Md * 3 * il_));
      R.o_d.push_back(alloc<bf16>(Md * il_));
      R.lse_d.push_back(alloc<float>(Md * hl_));
      R.ax_d.push_back(alloc<bf16>(Md * d_));
      if (fused_x_) {
        bf16* x = alloc<bf16>(Md * 3 * il_);
        R.cq_d.push_back(x);
        R.ckv_d.push_back(x + il_);
      } else {
        R.cq_d.push_back(alloc<bf16>(Md * il_));
        R.ckv_d.push_back(alloc<bf16>(Me * 2 * il_));
      }
      R.co_d.push_back(alloc<bf16>(Md * il_));
      R.clse_d.push_back(alloc<float>(Md * hl_));
      R.a2_d.push_back(alloc<bf16>(Md * d_));
      R.act_d.push_back(alloc<bf16>(Md * fl_));
    }
    R.stf_d = alloc<float>(Md);
    R.f = alloc<bf16>(Md * d_);
    R.logits = alloc<bf16>(Md * V_);
    R.ids_e = alloc<int32_t>(static_cast<int64_t>(Te_) * Te_);
    R.ids_d = alloc<int32_t>(static_cast<int64_t>(Td_) * Td_);
    cuda_check(cudaMemcpyAsync(R.ids_e, ids_e.data(), ids_e.size() * 4, cudaMemcpyHostToDevice, stream_), "H2D");
    cuda_check(cudaMemcpyAsync(R.ids_d, ids_d.data(), ids_d.size() * 4, cudaMemcpyHostToDevice, stream_), "H2D");
    if (tc_) {
      std::vector<int32_t> be(2 * static_cast<size_t>(Te_) - 1), bd(2 * static_cast<size_t>(Td_) - 1);
      for (int i = 0; i < 2 * Te_ - 1; ++i) be[i] = t5_rel_bucket(i - (Te_ - 1), true, nb_, maxd_);
      for (int i = 0; i < 2 * Td_ - 1; ++i) bd[i] = t5_rel_bucket(i - (Td_ - 1), false, nb_, maxd_);
      R.bd_e = alloc<int32_t>(static_cast<int64_t>(be.size()));
      R.bd_d = alloc<int32_t>(static_cast<int64_t>(bd.size()));
      cuda_check(cudaMemcpyAsync(R.bd_e, be.data(), be.size() * 4, cudaMemcpyHostToDevice, stream_), "H2D");
      cuda_check(cudaMemcpyAsync(R.bd_d, bd.data(), bd.size() * 4, cudaMemcpyHostToDevice, stream_), "H2D");
      R.lut_e = alloc<float>(static_cast<int64_t>(hl_) * (2 * Te_ + 128));
      R.dlut_e = alloc<float>(static_cast<int64_t>(hl_) * (2 * Te_ + 128));
      R.lut_d = alloc<float>(static_cast<int64_t>(hl_) * (2 * Td_ + 128));
      R.dlut_d = alloc<float>(static_cast<int64_t>(hl_) * (2 * Td_ + 128));
    } else {
      R.bias_e = alloc<float>(static_cast<int64_t>(hl_) * Te_ * Te_);
      R.dbias_e = alloc<float>(static_cast<int64_t>(hl_) * Te_ * Te_);
      R.bias_d = alloc<float>(static_cast<int64_t>(hl_) * Td_ * Td_);
      R.dbias_d = alloc<float>(static_cast<int64_t>(hl_) * Td_ * Td_);
    }
    R.enc_tok = alloc<int32_t>(Me);
    R.dec_tok = alloc<int32_t>(Md);
    R.targets = alloc<int32_t>(Md);
    R.weights = alloc<float>(Md);
    R.wloss = alloc<float>(Md);
    R.wsum = alloc<float>(1);
    R.loss = alloc<double>(1);
    R.gres_e = alloc<float>(Me * d_);
    R.gres_d = alloc<float>(Md * d_);
    R.dx = alloc<float>(Mx * d_);
    R.part = alloc<float>(Mx * d_);
    R.d_eout = alloc<float>(Me * d_);
    R.gb = alloc<bf16>(Mx * d_);
    R.dqkv = alloc<bf16>(Mx * 3 * il_);
    R.dout = alloc<bf16>(Mx * il_);
    R.dact = alloc<bf16>(Mx * fl_);
    R.dcq = alloc<bf16>(Md * il_);
    R.dckv = alloc<bf16>(Me * 2 * il_);
    const int Tx = Te_ > Td_ ? Te_ : Td_;
    R.attn_scratch = alloc<float>(k::t5_attention_scratch(B_, hl_, Tx, Tx, dk_));
    R.ln_partials = alloc<float>(k::layernorm_bwd_partials(d_));
    R.tok_keys = alloc<uint32_t>(k::embed_bwd_keys(Mx));
    ranks_.push_back(R);
  }
  d_flag_ = alloc<int>(1);
  cuda_check(cudaStreamSynchronize(stream_), "allocate");
}

// ---------------------------------------------------------------------------------------------
// parameters (the same materialiser rules as Model: contiguous even chunks, sharded_tensor.hpp)
// ---------------------------------------------------------------------------------------------
void T5Model::init_params(uint64_t seed, const std::string& stream_name) {
  poisoned_ = false;
  const uint64_t key = t5_mix64(seed ^ t5_mix64(t5_fnv1a(stream_name)));
  for (T5Rank& R : ranks_) {
    for (const Slot& s : slots_) {
      float* dst = R.p + s.offset;
      if (s.init == 1) {
        k::fill_f32(dst, s.numel, 1.0f, stream_);
      } else {
        int64_t r0 = 0, c0 = 0;
        if (s.layout.kind == Layout::kSplit) (s.layout.dim == 0 ? r0 : c0) = s.local[s.layout.dim] * R.mpi;
        k::init_normal(dst, s.local[0], s.local[1], r0, c0, s.global[1], key, s.draw_base, s.init_scale, stream_);
      }
      ++launches_;
    }
    cuda_check(cudaMemsetAsync(R.m, 0, flat_n_ * 4, stream_), "memset");
    cuda_check(cudaMemsetAsync(R.v, 0, flat_n_ * 4, stream_), "memset");
    k::cast_f32_bf16(R.p, R.w, flat_n_, stream_);
  }
  step_ = 0;
  cuda_check(cudaStreamSynchronize(stream_), "init_params");
}

void T5Model::set_tensor(const std::string& name, int which, const float* full, int64_t numel) {
  const auto it = slot_of_.find(name);
  if (it == slot_of_.end()) fail(SW_ERR_CONFIG, "TrainState: no parameter named '" + name + "'");
  const Slot& s = slots_[it->second];
  if (numel != t5_numel(s.global)) {
    fail(SW_ERR_SHAPE, "set_param: '" + name + "' expects " + std::to_string(t5_numel(s.global)) +
                           " elements, got " + std::to_string(numel));
  }
  if (which != 0 && which != 2 && which != 3) fail(SW_ERR_CONFIG, "set_tensor: `which` must be 0, 2 or 3");
  for (T5Rank& R : ranks_) {
    float* dst = (which == 0 ? R.p : which == 2 ? R.m : R.v) + s.offset;
    if (s.layout.kind != Layout::kSplit) {
      cuda_check(cudaMemcpyAsync(dst, full, numel * 4, cudaMemcpyHostToDevice, stream_), "H2D");
    } else if (s.layout.dim == 0) {
      const int64_t lr = s.local[0], cols = s.global[1];
      cuda_check(cudaMemcpyAsync(dst, full + R.mpi * lr * cols, lr * cols * 4, cudaMemcpyHostToDevice, stream_), "H2D");
    } else {
      const int64_t lc = s.local[1], rows = s.global[0], cols = s.global[1];
      cuda_check(cudaMemcpy2DAsync(dst, lc * 4, full + R.mpi * lc, cols * 4, lc * 4, rows, cudaMemcpyHostToDevice,
                                   stream_),
                 "H2D 2D");
    }
    if (which == 0) k::cast_f32_bf16(dst, R.w + s.offset, s.numel, stream_);
  }
  cuda_check(cudaStreamSynchronize(stream_), "set_param");
}

void T5Model::get_tensor(const std::string& name, int which, float* full, int64_t numel) {
  const auto it = slot_of_.find(name);
  if (it == slot_of_.end()) fail(SW_ERR_CONFIG, "TrainState: no parameter named '" + name + "'");
  const Slot& s = slots_[it->second];
  if (numel != t5_numel(s.global)) fail(SW_ERR_SHAPE, "get_tensor: '" + name + "' size mismatch");
  if (which < 0 || which > 3) fail(SW_ERR_CONFIG, "get_tensor: `which` must be 0..3");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  auto base = [&](T5Rank& R) { return (which == 0 ? R.p : which == 1 ? R.g : which == 2 ? R.m : R.v) + s.offset; };
  if (s.layout.kind != Layout::kSplit) {
    cuda_check(cudaMemcpy(full, base(ranks_[0]), numel * 4, cudaMemcpyDeviceToHost), "D2H");
    return;
  }
  const int64_t rows = s.global[0], cols = s.global[1];
  if (mesh_->emulated) {
    for (T5Rank& R : ranks_) {
      if (s.layout.dim == 0) {
        cuda_check(cudaMemcpy(full + R.mpi * s.local[0] * cols, base(R), s.numel * 4, cudaMemcpyDeviceToHost), "D2H");
      } else {
        const int64_t lc = s.local[1];
        cuda_check(cudaMemcpy2D(full + R.mpi * lc, cols * 4, base(R), lc * 4, lc * 4, rows, cudaMemcpyDeviceToHost),
                   "D2H 2D");
      }
    }
    return;
  }
  float* tmp = nullptr;
  cuda_check(cudaMalloc(&tmp, numel * 4), "cudaMalloc");
  nccl_check(ncclAllGather(base(ranks_[0]), tmp, s.numel, ncclFloat, mesh_->mp_comm, stream_), "AllGather");
  std::vector<float> host(static_cast<size_t>(numel));
  cuda_check(cudaMemcpyAsync(host.data(), tmp, numel * 4, cudaMemcpyDeviceToHost, stream_), "D2H");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  cudaFree(tmp);
  if (s.layout.dim == 0) {
    std::memcpy(full, host.data(), numel * 4);
  } else {
    const int64_t lc = s.local[1];
    for (int r = 0; r < mesh_->mp; ++r)
      for (int64_t i = 0; i < rows; ++i) std::memcpy(full + i * cols + r * lc, host.data() + r * s.numel + i * lc, lc * 4);
  }
}

void T5Model::stage_batch(const int32_t* enc, const int32_t* dec, const int32_t* targets, const float* weights) {
  for (T5Rank& R : ranks_) {
    cuda_check(cudaMemcpyAsync(R.enc_tok, enc, Me_ * 4, cudaMemcpyHostToDevice, stream_), "H2D");
    cuda_check(cudaMemcpyAsync(R.dec_tok, dec, Md_ * 4, cudaMemcpyHostToDevice, stream_), "H2D");
    cuda_check(cudaMemcpyAsync(R.targets, targets, Md_ * 4, cudaMemcpyHostToDevice, stream_), "H2D");
    if (weights != nullptr) {
      cuda_check(cudaMemcpyAsync(R.weights, weights, Md_ * 4, cudaMemcpyHostToDevice, stream_), "H2D");
    } else {
      k::fill_f32(R.weights, Md_, 1.0f, stream_);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// building blocks
// ---------------------------------------------------------------------------------------------
void T5Model::tic() {
  if (!prof_) return;
  if (ev_next_ + 2 > events_.size()) {
    for (int i = 0; i < 256; ++i) {
      cudaEvent_t e;
      cuda_check(cudaEventCreate(&e), "cudaEventCreate");
      events_.push_back(e);
    }
  }
  cuda_check(cudaEventRecord(events_[ev_next_], stream_), "cudaEventRecord");
}

void T5Model::toc(int cat, double work) {
  if (!prof_) return;
  cuda_check(cudaEventRecord(events_[ev_next_ + 1], stream_), "cudaEventRecord");
  ev_next_ += 2;
  prof_rec_.emplace_back(cat, work);
}

void T5Model::set_profiling(bool on) {
  prof_ = on;
  ev_next_ = 0;
  prof_rec_.clear();
}

void T5Model::read_profile(double* ms, double* work, int64_t* count) {
  for (int c = 0; c < kProfCats; ++c) ms[c] = work[c] = 0.0, count[c] = 0;
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  for (size_t i = 0; i < prof_rec_.size(); ++i) {
    float t = 0.f;
    cuda_check(cudaEventElapsedTime(&t, events_[2 * i], events_[2 * i + 1]), "cudaEventElapsedTime");
    ms[prof_rec_[i].first] += t;
    work[prof_rec_[i].first] += prof_rec_[i].second;
    count[prof_rec_[i].first] += 1;
  }
  ev_next_ = 0;
  prof_rec_.clear();
}

void T5Model::gemm(int M, int N, int K, const void* A, int64_t lda, int a_mn, const void* B, int64_t ldb, int b_mn,
                   int epi, void* C, int64_t ldc, const void* aux, int64_t ld_aux, int accumulate, int relu) {
  GemmParams p;
  p.relu = relu;
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
  p.aux = aux;
  p.ld_aux = ld_aux;
  p.accumulate = accumulate;
  tic();
  cuda_check(gemm_bf16(p, stream_), "gemm launch");
  toc(kProfGemm, 2.0 * M * N * static_cast<double>(K));
  ++launches_;
}

void T5Model::ar(const std::function<float*(T5Rank&)>& ptr, int64_t n) {
  if (mesh_->mp == 1) return;
  tic();
  if (mesh_->emulated) {
    std::vector<float*> ptrs;
    for (T5Rank& R : ranks_) ptrs.push_back(ptr(R));
    k::sum_ranks_f32(ptrs.data(), static_cast<int>(ptrs.size()), n, 1.0f, stream_);
    ++launches_;
  } else {
    nccl_check(ncclAllReduce(ptr(ranks_[0]), ptr(ranks_[0]), n, ncclFloat, ncclSum, mesh_->mp_comm, stream_),
               "AllReduce");
  }
  const double t = mesh_->mp;
  toc(kProfComm, 2.0 * (t - 1) / t * 4.0 * n);
  mesh_->record(CollKind::kAllReduce, mesh_->mp_group(0), static_cast<uint64_t>(n) * 4);
}

void T5Model::row_parallel(int64_t M, int K, const std::function<const bf16*(T5Rank&)>& a, int w_slot,
                           const std::function<const float*(T5Rank&)>& aux, const std::function<float*(T5Rank&)>& out) {
  if (t_ == 1) {
    for (T5Rank& R : ranks_) {
      gemm(static_cast<int>(M), d_, K, a(R), K, 0, W(R, w_slot), K, 0, static_cast<int>(Epi::kResidF32), out(R), d_,
           aux(R), d_);
    }
    return;
  }
  for (T5Rank& R : ranks_) {
    gemm(static_cast<int>(M), d_, K, a(R), K, 0, W(R, w_slot), K, 0, static_cast<int>(Epi::kStoreF32), R.part, d_);
  }
  ar([](T5Rank& R) { return R.part; }, M * d_);
  for (T5Rank& R : ranks_) {
    k::add_residual_bias(aux(R), R.part, nullptr, out(R), M, d_, stream_);
    ++launches_;
  }
}

void T5Model::attn_fwd(T5Rank& R, int Tq, int Tk, const bf16* q, int64_t ldq, const bf16* kp, const bf16* vp,
                       int64_t ldkv, bf16* o, float* lse, const float* bias, int causal) {
  k::T5AttnArgs a;
  a.q = q;
  a.ldq = ldq;
  a.k = kp;
  a.ldk = ldkv;
  a.v = vp;
  a.ldv = ldkv;
  a.o = o;
  a.ldo = il_;
  a.lse = lse;
  a.bias = bias;
  a.Tq = Tq;
  a.Tk = Tk;
  a.Hl = hl_;
  a.dk = dk_;
  a.causal = causal;
  a.scale = 1.0f;  // T5: no 1/sqrt(d_kv)
  (void)R;
  tic();
  // tcgen05 path: fused q|k|v rows (ld 3*inner/t, k and v at +inner/t, +2*inner/t), Tq == Tk
  const bool tc = tc_ && Tq == Tk && ldq == 3LL * il_ && ldkv == 3LL * il_ && kp == q + il_ && vp == q + 2 * il_;
  const bool tc_cross = tc_ && !tc && bias == nullptr && !causal;  // separate q and encoder k|v rows
  if (!(tc && k::attention_fwd_ex(q, o, lse, B_, Tq, hl_, dk_, causal, bias, 1.0f, stream_)) &&
      !(tc_cross && k::attention_fwd_cross(q, ldq, kp, ldkv, static_cast<int>(vp - kp), o, lse, B_, Tq, Tk, hl_, dk_,
                                           1.0f, stream_))) {
    if (tc_ && bias != nullptr) fail(SW_ERR_INTERNAL, "T5: the tcgen05 attention forward declined a biased self-attention");
    k::t5_attention_fwd(a, B_, stream_);
  }
  toc(kProfAttnFwd, 4.0 * B_ * hl_ * static_cast<double>(Tq) * Tk * dk_ * (causal ? 0.5 : 1.0));
  ++launches_;
}

void T5Model::rms_fwd(const float* x, int scale_slot, T5Rank& R, bf16* y, float* rstd, int64_t M) {
  tic();
  k::layernorm_fwd(x, P(R, scale_slot), nullptr, y, nullptr, rstd, M, d_, kT5Eps, stream_, 1);
  toc(kProfNorm, 6.0 * M * d_);
  ++launches_;
}

void T5Model::rms_bwd(const float* x, const float* rstd, int scale_slot, T5Rank& R, const float* dy, float* gres,
                      int64_t M, int accumulate) {
  tic();
  k::layernorm_bwd(x, nullptr, rstd, P(R, scale_slot), dy, gres, R.gb, G(R, scale_slot), nullptr, M, d_, accumulate,
                   stream_, R.ln_partials, 1);
  toc(kProfNorm, 18.0 * M * d_);
  ++launches_;
}

// ---------------------------------------------------------------------------------------------
// forward (oracle/t5_ref.py forward_backward, first half)
// ---------------------------------------------------------------------------------------------
void T5Model::forward(bool need_grad) {
  cuda_check(cudaSetDevice(mesh_->cuda_device), "cudaSetDevice");
  const int64_t Me = Me_, Md = Md_;
  const int d = d_, il = il_, fl = fl_;
  for (T5Rank& R : ranks_) {
    const int h0 = R.mpi * hl_;
    if (tc_) {
      k::t5_lut_build(P(R, rb_e_), R.bd_e, H_, h0, hl_, Te_, R.lut_e, stream_);
      k::t5_lut_build(P(R, rb_d_), R.bd_d, H_, h0, hl_, Td_, R.lut_d, stream_);
    } else {
      k::t5_bias_build(P(R, rb_e_), R.ids_e, H_, h0, hl_, static_cast<int64_t>(Te_) * Te_, R.bias_e, stream_);
      k::t5_bias_build(P(R, rb_d_), R.ids_d, H_, h0, hl_, static_cast<int64_t>(Td_) * Td_, R.bias_d, stream_);
    }
    k::embed_fwd(R.enc_tok, P(R, tok_), nullptr, R.hs_e[0], Me, Te_, d, stream_);
    k::embed_fwd(R.dec_tok, P(R, tok_), nullptr, R.hs_d[0], Md, Td_, d, stream_);
    launches_ += 4;
  }
  // ---- encoder ----
  for (int l = 0; l < Le_; ++l) {
    const T5Layer& L = enc_[l];
    for (T5Rank& R : ranks_) {
      rms_fwd(R.hs_e[l], L.ln1, R, R.a1_e[l], R.st1_e[l], Me);
      gemm(static_cast<int>(Me), 3 * il, d, R.a1_e[l], d, 0, W(R, L.q), d, 0, static_cast<int>(Epi::kStoreBf16),
           R.qkv_e[l], 3 * il);
      attn_fwd(R, Te_, Te_, R.qkv_e[l], 3 * il, R.qkv_e[l] + il, R.qkv_e[l] + 2 * il, 3 * il, R.o_e[l], R.lse_e[l],
               tc_ ? R.lut_e : R.bias_e, 0);
    }
    row_parallel(Me, il, [&](T5Rank& R) -> const bf16* { return R.o_e[l]; }, L.o,
                 [&](T5Rank& R) -> const float* { return R.hs_e[l]; }, [&](T5Rank& R) { return R.hm_e[l]; });
    for (T5Rank& R : ranks_) {
      rms_fwd(R.hm_e[l], L.ln2, R, R.a2_e[l], R.st2_e[l], Me);
      gemm(static_cast<int>(Me), fl, d, R.a2_e[l], d, 0, W(R, L.fc1), d, 0, static_cast<int>(Epi::kStoreBf16),
           R.act_e[l], fl, nullptr, 0, 0, /*relu=*/1);
    }
    row_parallel(Me, fl, [&](T5Rank& R) -> const bf16* { return R.act_e[l]; }, L.fc2,
                 [&](T5Rank& R) -> const float* { return R.hm_e[l]; }, [&](T5Rank& R) { return R.hs_e[l + 1]; });
  }
  for (T5Rank& R : ranks_) rms_fwd(R.hs_e[Le_], lnf_e_, R, R.eo, R.stf_e, Me);
  // ---- decoder ----
  for (int l = 0; l < Ld_; ++l) {
    const T5Layer& L = dec_[l];
    for (T5Rank& R : ranks_) {
      rms_fwd(R.hs_d[l], L.ln1, R, R.a1_d[l], R.st1_d[l], Md);
      gemm(static_cast<int>(Md), 3 * il, d, R.a1_d[l], d, 0, W(R, L.q), d, 0, static_cast<int>(Epi::kStoreBf16),
           R.qkv_d[l], 3 * il);
      attn_fwd(R, Td_, Td_, R.qkv_d[l], 3 * il, R.qkv_d[l] + il, R.qkv_d[l] + 2 * il, 3 * il, R.o_d[l], R.lse_d[l],
               tc_ ? R.lut_d : R.bias_d, 1);
    }
    row_parallel(Md, il, [&](T5Rank& R) -> const bf16* { return R.o_d[l]; }, L.o,
                 [&](T5Rank& R) -> const float* { return R.hs_d[l]; }, [&](T5Rank& R) { return R.hm_d[l]; });
    for (T5Rank& R : ranks_) {
      rms_fwd(R.hm_d[l], L.lnx, R, R.ax_d[l], R.stx_d[l], Md);
      gemm(static_cast<int>(Md), il, d, R.ax_d[l], d, 0, W(R, L.cq), d, 0, static_cast<int>(Epi::kStoreBf16),
           R.cq_d[l], ld_cq_);
      gemm(static_cast<int>(Me), 2 * il, d, R.eo, d, 0, W(R, L.ck), d, 0, static_cast<int>(Epi::kStoreBf16),
           R.ckv_d[l], ld_ckv_);
      attn_fwd(R, Td_, Te_, R.cq_d[l], ld_cq_, R.ckv_d[l], R.ckv_d[l] + il, ld_ckv_, R.co_d[l], R.clse_d[l], nullptr,
               0);
    }
    row_parallel(Md, il, [&](T5Rank& R) -> const bf16* { return R.co_d[l]; }, L.co,
                 [&](T5Rank& R) -> const float* { return R.hm_d[l]; }, [&](T5Rank& R) { return R.hx_d[l]; });
    for (T5Rank& R : ranks_) {
      rms_fwd(R.hx_d[l], L.ln2, R, R.a2_d[l], R.st2_d[l], Md);
      gemm(static_cast<int>(Md), fl, d, R.a2_d[l], d, 0, W(R, L.fc1), d, 0, static_cast<int>(Epi::kStoreBf16),
           R.act_d[l], fl, nullptr, 0, 0, /*relu=*/1);
    }
    row_parallel(Md, fl, [&](T5Rank& R) -> const bf16* { return R.act_d[l]; }, L.fc2,
                 [&](T5Rank& R) -> const float* { return R.hx_d[l]; }, [&](T5Rank& R) { return R.hs_d[l + 1]; });
  }
  for (T5Rank& R : ranks_) {
    rms_fwd(R.hs_d[Ld_], lnf_d_, R, R.f, R.stf_d, Md);
    gemm(static_cast<int>(Md), V_, d, R.f, d, 0, W(R, head_), d, 0, static_cast<int>(Epi::kStoreBf16), R.logits, V_);
    k::sum_f32(R.weights, Md, R.wsum, stream_);
    tic();
    k::xent_fwd_bwd(R.logits, V_, Md, V_, R.targets, R.weights, R.wsum, R.wloss, need_grad ? 1 : 0, stream_);
    toc(kProfXent, (need_grad ? 4.0 : 2.0) * Md * V_);
    k::loss_reduce(R.wloss, Md, R.wsum, R.loss, stream_, fused_ != nullptr ? d_flag_ : nullptr);
    launches_ += 3;
  }
}

// ---------------------------------------------------------------------------------------------
// backward (oracle/t5_ref.py forward_backward, second half)
// ---------------------------------------------------------------------------------------------
void T5Model::backward() {
  const int64_t Me = Me_, Md = Md_;
  const int d = d_, il = il_, fl = fl_;
  const int F32 = static_cast<int>(Epi::kStoreF32), BF = static_cast<int>(Epi::kStoreBf16);
  for (T5Rank& R : ranks_) {
    cuda_check(cudaMemsetAsync(R.g, 0, flat_n_ * 4, stream_), "memset");
    if (tc_) {
      cuda_check(cudaMemsetAsync(R.dlut_e, 0, sizeof(float) * hl_ * (2 * Te_ + 128), stream_), "memset");
      cuda_check(cudaMemsetAsync(R.dlut_d, 0, sizeof(float) * hl_ * (2 * Td_ + 128), stream_), "memset");
    } else {
      cuda_check(cudaMemsetAsync(R.dbias_e, 0, sizeof(float) * hl_ * Te_ * Te_, stream_), "memset");
      cuda_check(cudaMemsetAsync(R.dbias_d, 0, sizeof(float) * hl_ * Td_ * Td_, stream_), "memset");
    }
    cuda_check(cudaMemsetAsync(R.d_eout, 0, sizeof(float) * Me * d, stream_), "memset");
    // d(final) = dlogits . W_head; dW_head = dlogits^T . f (replicated head: no collective)
    gemm(static_cast<int>(Md), d, V_, R.logits, V_, 0, W(R, head_), d, 1, F32, R.dx, d);
    wgrad(R, head_, V_, d, static_cast<int>(Md), R.logits, V_, R.f, d);
    rms_bwd(R.hs_d[Ld_], R.stf_d, lnf_d_, R, R.dx, R.gres_d, Md, 0);
  }
  auto attn_bwd = [&](T5Rank& R, int Tq, int Tk, const bf16* q, int64_t ldq, const bf16* kp, const bf16* vp,
                      int64_t ldkv, const bf16* o, const float* lse, const float* bias, int causal, bf16* dq,
                      int64_t lddq, bf16* dkp, bf16* dvp, int64_t lddkv, float* dbias) {
    k::T5AttnArgs a;
    a.q = q;
    a.ldq = ldq;
    a.k = kp;
    a.ldk = ldkv;
    a.v = vp;
    a.ldv = ldkv;
    a.o = const_cast<bf16*>(o);
    a.ldo = il;
    a.lse = const_cast<float*>(lse);
    a.bias = bias;
    a.Tq = Tq;
    a.Tk = Tk;
    a.Hl = hl_;
    a.dk = dk_;
    a.causal = causal;
    a.scale = 1.0f;
    tic();
    const bool tc = tc_ && Tq == Tk && ldq == 3LL * il && ldkv == 3LL * il && kp == q + il && vp == q + 2 * il &&
                    lddq == 3LL * il && lddkv == 3LL * il && dkp == dq + il && dvp == dq + 2 * il;
    const bool tc_cross = tc_ && !tc && bias == nullptr && !causal && vp - kp == dvp - dkp;
    if (!(tc && k::attention_bwd_ex(q, o, lse, R.dout, dq, R.attn_scratch, B_, Tq, hl_, dk_, causal, bias, dbias, 1.0f,
                                    stream_)) &&
        !(tc_cross && k::attention_bwd_cross(q, ldq, kp, ldkv, static_cast<int>(vp - kp), o, lse, R.dout, dq, lddq, dkp,
                                             lddkv, R.attn_scratch, B_, Tq, Tk, hl_, dk_, 1.0f, stream_))) {
      if (tc_ && bias != nullptr) fail(SW_ERR_INTERNAL, "T5: the tcgen05 attention backward declined (SW_ATTN_BWD_V1?)");
      k::t5_attention_bwd(a, B_, R.dout, il, dq, lddq, dkp, lddkv, dvp, lddkv, R.attn_scratch, dbias, stream_);
    }
    toc(kProfAttnBwd, 8.0 * B_ * hl_ * static_cast<double>(Tq) * Tk * dk_ * (causal ? 0.5 : 1.0));
    launches_ += 3;
  };
  // ---- decoder, last layer first ----
  for (int l = Ld_ - 1; l >= 0; --l) {
    const T5Layer& L = dec_[l];
    // MLP
    for (T5Rank& R : ranks_) {
      gemm(static_cast<int>(Md), fl, d, R.gb, d, 0, W(R, L.fc2), fl, 1, static_cast<int>(Epi::kGeluBwd), R.dact, fl,
           R.act_d[l], fl, 0, /*relu=*/1);
      wgrad(R, L.fc2, d, fl, static_cast<int>(Md), R.gb, d, R.act_d[l], fl);
      gemm(static_cast<int>(Md), d, fl, R.dact, fl, 0, W(R, L.fc1), d, 1, F32, R.dx, d);
      wgrad(R, L.fc1, fl, d, static_cast<int>(Md), R.dact, fl, R.a2_d[l], d);
    }
    ar([](T5Rank& R) { return R.dx; }, Md * d);
    for (T5Rank& R : ranks_) rms_bwd(R.hx_d[l], R.st2_d[l], L.ln2, R, R.dx, R.gres_d, Md, 1);
    // cross attention
    for (T5Rank& R : ranks_) {
      gemm(static_cast<int>(Md), il, d, R.gb, d, 0, W(R, L.co), il, 1, BF, R.dout, il);
      wgrad(R, L.co, d, il, static_cast<int>(Md), R.gb, d, R.co_d[l], il);
      // fused layout: dq | dk | dv land in one [M, 3*inner/t] buffer like the forward's
      bf16* dcq = fused_x_ ? R.dqkv : R.dcq;
      bf16* dckv = fused_x_ ? R.dqkv + il : R.dckv;
      attn_bwd(R, Td_, Te_, R.cq_d[l], ld_cq_, R.ckv_d[l], R.ckv_d[l] + il, ld_ckv_, R.co_d[l], R.clse_d[l], nullptr, 0,
               dcq, ld_cq_, dckv, dckv + il, ld_ckv_, nullptr);
      gemm(static_cast<int>(Md), d, il, dcq, ld_cq_, 0, W(R, L.cq), d, 1, F32, R.dx, d);
      wgrad(R, L.cq, il, d, static_cast<int>(Md), dcq, ld_cq_, R.ax_d[l], d);
      // encoder-output gradient: partial over the mp group, summed over layers, reduced once
      gemm(static_cast<int>(Me), d, 2 * il, dckv, ld_ckv_, 0, W(R, L.ck), d, 1, F32, R.d_eout, d, nullptr, 0, 1);
      wgrad(R, L.ck, 2 * il, d, static_cast<int>(Me), dckv, ld_ckv_, R.eo, d);
    }
    ar([](T5Rank& R) { return R.dx; }, Md * d);
    for (T5Rank& R : ranks_) rms_bwd(R.hm_d[l], R.stx_d[l], L.lnx, R, R.dx, R.gres_d, Md, 1);
    // self attention (causal, relative bias)
    for (T5Rank& R : ranks_) {
      gemm(static_cast<int>(Md), il, d, R.gb, d, 0, W(R, L.o), il, 1, BF, R.dout, il);
      wgrad(R, L.o, d, il, static_cast<int>(Md), R.gb, d, R.o_d[l], il);
      attn_bwd(R, Td_, Td_, R.qkv_d[l], 3 * il, R.qkv_d[l] + il, R.qkv_d[l] + 2 * il, 3 * il, R.o_d[l], R.lse_d[l],
               tc_ ? R.lut_d : R.bias_d, 1, R.dqkv, 3 * il, R.dqkv + il, R.dqkv + 2 * il, 3 * il,
               tc_ ? R.dlut_d : R.dbias_d);
      gemm(static_cast<int>(Md), d, 3 * il, R.dqkv, 3 * il, 0, W(R, L.q), d, 1, F32, R.dx, d);
      wgrad(R, L.q, 3 * il, d, static_cast<int>(Md), R.dqkv, 3 * il, R.a1_d[l], d);
    }
    ar([](T5Rank& R) { return R.dx; }, Md * d);
    for (T5Rank& R : ranks_) rms_bwd(R.hs_d[l], R.st1_d[l], L.ln1, R, R.dx, R.gres_d, Md, 1);
  }
  for (T5Rank& R : ranks_) {
    k::embed_bwd_tok(R.dec_tok, R.gres_d, G(R, tok_), Md, d, V_, R.tok_keys, stream_);
    if (tc_)
      k::t5_lut_grad(R.dlut_d, R.bd_d, H_, R.mpi * hl_, hl_, Td_, G(R, rb_d_), stream_);
    else
      k::t5_bias_grad(R.dbias_d, R.ids_d, H_, R.mpi * hl_, hl_, static_cast<int64_t>(Td_) * Td_, nb_, G(R, rb_d_),
                      stream_);
    launches_ += 2;
  }
  ar([this](T5Rank& R) { return G(R, rb_d_); }, static_cast<int64_t>(nb_) * H_);
  // ---- encoder ----
  ar([](T5Rank& R) { return R.d_eout; }, Me * d);
  for (T5Rank& R : ranks_) rms_bwd(R.hs_e[Le_], R.stf_e, lnf_e_, R, R.d_eout, R.gres_e, Me, 0);
  for (int l = Le_ - 1; l >= 0; --l) {
    const T5Layer& L = enc_[l];
    for (T5Rank& R : ranks_) {
      // dact = (gb . W_fc2) * relu'(act), the ReLU derivative from the stored activation
      gemm(static_cast<int>(Me), fl, d, R.gb, d, 0, W(R, L.fc2), fl, 1, static_cast<int>(Epi::kGeluBwd), R.dact, fl,
           R.act_e[l], fl, 0, /*relu=*/1);
      wgrad(R, L.fc2, d, fl, static_cast<int>(Me), R.gb, d, R.act_e[l], fl);
      gemm(static_cast<int>(Me), d, fl, R.dact, fl, 0, W(R, L.fc1), d, 1, F32, R.dx, d);
      wgrad(R, L.fc1, fl, d, static_cast<int>(Me), R.dact, fl, R.a2_e[l], d);
    }
    ar([](T5Rank& R) { return R.dx; }, Me * d);
    for (T5Rank& R : ranks_) rms_bwd(R.hm_e[l], R.st2_e[l], L.ln2, R, R.dx, R.gres_e, Me, 1);
    for (T5Rank& R : ranks_) {
      gemm(static_cast<int>(Me), il, d, R.gb, d, 0, W(R, L.o), il, 1, BF, R.dout, il);
      wgrad(R, L.o, d, il, static_cast<int>(Me), R.gb, d, R.o_e[l], il);
      attn_bwd(R, Te_, Te_, R.qkv_e[l], 3 * il, R.qkv_e[l] + il, R.qkv_e[l] + 2 * il, 3 * il, R.o_e[l], R.lse_e[l],
               tc_ ? R.lut_e : R.bias_e, 0, R.dqkv, 3 * il, R.dqkv + il, R.dqkv + 2 * il, 3 * il,
               tc_ ? R.dlut_e : R.dbias_e);
      gemm(static_cast<int>(Me), d, 3 * il, R.dqkv, 3 * il, 0, W(R, L.q), d, 1, F32, R.dx, d);
      wgrad(R, L.q, 3 * il, d, static_cast<int>(Me), R.dqkv, 3 * il, R.a1_e[l], d);
    }
    ar([](T5Rank& R) { return R.dx; }, Me * d);
    for (T5Rank& R : ranks_) rms_bwd(R.hs_e[l], R.st1_e[l], L.ln1, R, R.dx, R.gres_e, Me, 1);
  }
  for (T5Rank& R : ranks_) {
    k::embed_bwd_tok(R.enc_tok, R.gres_e, G(R, tok_), Me, d, V_, R.tok_keys, stream_);
    if (tc_)
      k::t5_lut_grad(R.dlut_e, R.bd_e, H_, R.mpi * hl_, hl_, Te_, G(R, rb_e_), stream_);
    else
      k::t5_bias_grad(R.dbias_e, R.ids_e, H_, R.mpi * hl_, hl_, static_cast<int64_t>(Te_) * Te_, nb_, G(R, rb_e_),
                      stream_);
    launches_ += 2;
  }
  ar([this](T5Rank& R) { return G(R, rb_e_); }, static_cast<int64_t>(nb_) * H_);
}

void T5Model::forward_backward() {
  check_not_poisoned("t5 forward_backward");
  launches_ = 0;
  forward(true);
  backward();
  cuda_check(cudaGetLastError(), "t5 forward_backward");
}

void T5Model::forward_only() {
  forward(false);
  cuda_check(cudaGetLastError(), "t5 forward");
}

void T5Model::adamw(double lr, double b1, double b2, double eps, double wd) {
  check_not_poisoned("t5 adamw_step");
  const double t = static_cast<double>(step_ + 1);
  const float c1 = static_cast<float>(1.0 - std::pow(b1, t));
  const float c2 = static_cast<float>(1.0 - std::pow(b2, t));
  for (T5Rank& R : ranks_) {
    tic();
    k::adamw(R.p, R.m, R.v, R.g, R.w, flat_n_, static_cast<float>(lr), static_cast<float>(b1), static_cast<float>(b2),
             static_cast<float>(eps), static_cast<float>(wd), c1, c2, stream_);
    toc(kProfAdamw, 30.0 * flat_n_);
    ++launches_;
  }
  ++step_;
  cuda_check(cudaGetLastError(), "t5 adamw");
}

void T5Model::wgrad(T5Rank& R, int slot, int M, int N, int K, const void* A, int64_t lda, const void* B,
                    int64_t ldb) {
  if (fused_ == nullptr || slots_[slot].offset >= weights_end_) {
    gemm(M, N, K, A, lda, 1, B, ldb, 1, static_cast<int>(Epi::kStoreF32), G(R, slot), N);
    return;
  }
  // optimizer in the epilogue (as Model::wgrad): the gradient never leaves the accumulator
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
  ++launches_;
}

void T5Model::check_not_poisoned(const char* what) const {
  if (poisoned_) {
    fail(SW_ERR_NONFINITE, std::string(what) + ": a fused step found a non-finite gradient after updating some "
                                               "weights; re-initialise the model (init_params)");
  }
}

bool T5Model::train_step(double lr, double b1, double b2, double eps, double wd) {
  check_not_poisoned("t5 train_step");
  static const bool disabled = [] {
    const char* e = std::getenv("SW_FUSED_ADAMW");
    return e != nullptr && e[0] == '0';
  }();
  if (disabled) {
    forward_backward();
    adamw(lr, b1, b2, eps, wd);
    return false;
  }
  // Optimizer in the backward: every GEMM weight is updated by its wgrad epilogue (each weight's
  // dgrad, which reads the bf16 shadow, is issued before its wgrad), the region-2 parameters by
  // one flat AdamW after the backward. A non-finite loss gates every fused update.
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
    forward_backward();
  } catch (...) {
    fused_ = nullptr;
    throw;
  }
  fused_ = nullptr;
  int flag = 0;
  cuda_check(cudaMemcpyAsync(&flag, d_flag_, sizeof(int), cudaMemcpyDeviceToHost, stream_), "D2H");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  if (flag & 2) fail(SW_ERR_NONFINITE, "t5 train_step: non-finite loss; no parameter was updated");
  if (flag) {
    poisoned_ = true;
    fail(SW_ERR_NONFINITE, "t5 train_step: non-finite gradient (optimizer fused into the backward: the GEMM "
                           "weights updated before it was found keep their update; the model refuses further "
                           "steps until init_params)");
  }
  const int64_t n_small = flat_n_ - weights_end_;
  for (T5Rank& R : ranks_) {
    tic();
    k::adamw(R.p + weights_end_, R.m + weights_end_, R.v + weights_end_, R.g + weights_end_, R.w + weights_end_,
             n_small, fa.lr, fa.b1, fa.b2, fa.eps, fa.wd, fa.c1, fa.c2, stream_);
    toc(kProfAdamw, 30.0 * n_small);
    ++launches_;
  }
  ++step_;
  cuda_check(cudaGetLastError(), "t5 train_step");
  return true;
}

double T5Model::last_loss() {
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  double x = 0.0;
  cuda_check(cudaMemcpy(&x, ranks_[0].loss, sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  return x;
}

void T5Model::logits_to_host(float* out) {
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  std::vector<bf16> tmp(static_cast<size_t>(Md_) * V_);
  cuda_check(cudaMemcpy(tmp.data(), ranks_[0].logits, tmp.size() * 2, cudaMemcpyDeviceToHost), "D2H");
  for (size_t i = 0; i < tmp.size(); ++i) out[i] = __bfloat162float(tmp[i]);
}

}  // namespace sw
