// C ABI of the mesh and the model program / train state (include/shardweave_b200.h).
#include <cstring>
#include <string>

#include "mesh.h"
#include "model.h"
#include "t5.h"
#include "status.h"

struct sw_model_spec {
  sw::ModelSpec spec;
};
struct sw_plan {
  sw::Plan plan;
};
struct sw_mesh {
  sw::Mesh* mesh;
};
struct sw_model {
  sw::Model* model;
};
struct sw_t5 {
  sw::T5Model* model;
};

namespace {

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (p == nullptr) sw::fail(SW_ERR_INTERNAL, "out of host memory");
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

template <typename T>
void require(const T* p, const char* what) {
  if (p == nullptr) sw::fail(SW_ERR_CONFIG, std::string(what) + " is NULL");
}

}  // namespace

extern "C" {

sw_status sw_nccl_unique_id(uint8_t out[128]) {
  return sw::guarded([&] {
    ncclUniqueId id;
    sw::nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, sizeof(id));
  });
}

sw_status sw_mesh_create(int dp, int mp, int n_hosts, int rank, int world, const uint8_t* nccl_id,
                         int cuda_device, sw_mesh** out) {
  return sw::guarded([&] {
    require(out, "out");
    *out = new sw_mesh{sw::create_mesh(dp, mp, n_hosts, rank, world, nccl_id, cuda_device)};
  });
}

sw_status sw_mesh_comm_report(const sw_mesh* mesh, char** csv_out) {
  return sw::guarded([&] {
    require(mesh, "mesh");
    *csv_out = dup_string(mesh->mesh->report_csv());
  });
}

sw_status sw_mesh_reset_comm_report(sw_mesh* mesh) {
  return sw::guarded([&] {
    require(mesh, "mesh");
    for (auto& s : mesh->mesh->stats) s = sw::CommStat{};
  });
}

void sw_mesh_free(sw_mesh* mesh) {
  if (mesh != nullptr) {
    delete mesh->mesh;
    delete mesh;
  }
}

sw_status sw_model_create(const sw_model_spec* spec, const sw_plan* plan, sw_mesh* mesh, int batch,
                          int seq_len, sw_model** out) {
  return sw::guarded([&] {
    require(spec, "spec");
    require(plan, "plan");
    require(mesh, "mesh");
    require(out, "out");
    *out = new sw_model{new sw::Model(spec->spec, plan->plan, mesh->mesh, batch, seq_len)};
  });
}

sw_status sw_model_create_inference(const sw_model_spec* spec, const sw_plan* plan, sw_mesh* mesh, int batch,
                                    int seq_len, sw_model** out) {
  return sw::guarded([&] {
    require(spec, "spec");
    require(plan, "plan");
    require(mesh, "mesh");
    require(out, "out");
    *out = new sw_model{new sw::Model(spec->spec, plan->plan, mesh->mesh, batch, seq_len, true)};
  });
}

void sw_model_free(sw_model* model) {
  if (model != nullptr) {
    delete model->model;
    delete model;
  }
}

sw_status sw_model_init_params(sw_model* model, uint64_t seed, const char* stream_name) {
  return sw::guarded([&] {
    require(model, "model");
    model->model->init_params(seed, stream_name != nullptr ? stream_name : "model-init");
  });
}

sw_status sw_model_set_param(sw_model* model, const char* name, const float* full, int64_t numel) {
  return sw::guarded([&] {
    require(model, "model");
    require(name, "name");
    require(full, "full");
    model->model->set_param(name, full, numel);
  });
}

sw_status sw_model_get_tensor(sw_model* model, const char* name, int which, float* full_out,
                              int64_t numel) {
  return sw::guarded([&] {
    require(model, "model");
    require(name, "name");
    require(full_out, "full_out");
    model->model->get_tensor(name, which, full_out, numel);
  });
}

sw_status sw_model_stage_batch(sw_model* model, const int32_t* tokens, const int32_t* targets,
                               const float* weights) {
  return sw::guarded([&] {
    require(model, "model");
    require(tokens, "tokens");
    require(targets, "targets");
    model->model->stage_batch(tokens, targets, weights);
  });
}

sw_status sw_model_forward_backward(sw_model* model, int accumulate) {
  return sw::guarded([&] {
    require(model, "model");
    model->model->forward_backward(accumulate != 0);
  });
}

sw_status sw_model_scale_grads(sw_model* model, double factor) {
  return sw::guarded([&] {
    require(model, "model");
    model->model->scale_grads(factor);
  });
}

sw_status sw_model_dp_sync(sw_model* model) {
  return sw::guarded([&] {
    require(model, "model");
    model->model->dp_sync();
  });
}

sw_status sw_model_adamw_step(sw_model* model, const sw_adamw_cfg* cfg, int check_finite) {
  return sw::guarded([&] {
    require(model, "model");
    require(cfg, "cfg");
    model->model->adamw(cfg->lr, cfg->beta1, cfg->beta2, cfg->eps, cfg->weight_decay, check_finite != 0);
  });
}

sw_status sw_model_train_step(sw_model* model, const sw_adamw_cfg* cfg) {
  return sw::guarded([&] {
    require(model, "model");
    require(cfg, "cfg");
    model->model->train_step(cfg->lr, cfg->beta1, cfg->beta2, cfg->eps, cfg->weight_decay);
  });
}

sw_status sw_model_last_loss(sw_model* model, double* loss_out) {
  return sw::guarded([&] {
    require(model, "model");
    require(loss_out, "loss_out");
    *loss_out = model->model->last_loss();
  });
}

sw_status sw_model_forward_logits(sw_model* model, float* logits_out) {
  return sw::guarded([&] {
    require(model, "model");
    require(logits_out, "logits_out");
    model->model->forward_only();
    model->model->logits_to_host(logits_out);
  });
}

sw_status sw_model_stream(sw_model* model, void** stream_out) {
  return sw::guarded([&] {
    require(model, "model");
    *stream_out = model->model->stream();
  });
}

sw_status sw_model_launch_count(sw_model* model, int64_t* out) {
  return sw::guarded([&] {
    require(model, "model");
    *out = model->model->launches();
  });
}

sw_status sw_model_set_profiling(sw_model* model, int enable) {
  return sw::guarded([&] {
    require(model, "model");
    model->model->set_profiling(enable != 0);
  });
}

sw_status sw_model_read_profile(sw_model* model, double ms[8], double work[8], int64_t count[8]) {
  return sw::guarded([&] {
    require(model, "model");
    model->model->read_profile(ms, work, count);
  });
}

sw_status sw_model_device_bytes(sw_model* model, int64_t* out) {
  return sw::guarded([&] {
    require(model, "model");
    *out = model->model->device_bytes();
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// SWCK snapshots
// ---------------------------------------------------------------------------------------------
struct sw_checkpoint {
  sw::Checkpoint ck;
};

namespace {
std::vector<sw::CkptRng> rng_list(uint32_t n, const char* const* names, const uint64_t* seeds, const uint64_t* ids,
                                  const uint64_t* counters) {
  std::vector<sw::CkptRng> out;
  if (n > 0) {
    require(names, "rng_names");
    require(seeds, "rng_seeds");
    require(ids, "rng_stream_ids");
    require(counters, "rng_counters");
  }
  for (uint32_t i = 0; i < n; ++i) {
    require(names[i], "rng name");
    out.push_back(sw::CkptRng{names[i], seeds[i], ids[i], counters[i]});
  }
  return out;
}
}  // namespace

extern "C" {

sw_status sw_model_generate(sw_model* model, const int32_t* prompts, int P, int n_new, int32_t* out) {
  return sw::guarded([&] {
    require(model, "model");
    require(prompts, "prompts");
    require(out, "out");
    model->model->generate(prompts, P, n_new, out);
  });
}

sw_status sw_model_save_checkpoint(sw_model* model, const char* path, uint32_t n_rngs, const char* const* rng_names,
                                   const uint64_t* rng_seeds, const uint64_t* rng_stream_ids,
                                   const uint64_t* rng_counters) {
  return sw::guarded([&] {
    require(model, "model");
    require(path, "path");
    model->model->save_checkpoint(path, rng_list(n_rngs, rng_names, rng_seeds, rng_stream_ids, rng_counters));
  });
}

sw_status sw_model_load_checkpoint(sw_model* model, const char* path, uint32_t* n_rngs_out) {
  return sw::guarded([&] {
    require(model, "model");
    require(path, "path");
    model->model->load_checkpoint(path);
    if (n_rngs_out != nullptr) *n_rngs_out = static_cast<uint32_t>(model->model->loaded_rngs().size());
  });
}

sw_status sw_model_checkpoint_rng(sw_model* model, uint32_t index, char* name, uint64_t name_cap, uint64_t* seed,
                                  uint64_t* stream_id, uint64_t* counter) {
  return sw::guarded([&] {
    require(model, "model");
    const auto& r = model->model->loaded_rngs();
    if (index >= r.size()) sw::fail(SW_ERR_CONFIG, "checkpoint rng index out of range");
    if (name != nullptr) {
      if (name_cap < r[index].name.size() + 1) sw::fail(SW_ERR_CONFIG, "checkpoint rng name buffer too small");
      std::memcpy(name, r[index].name.c_str(), r[index].name.size() + 1);
    }
    if (seed) *seed = r[index].seed;
    if (stream_id) *stream_id = r[index].stream_id;
    if (counter) *counter = r[index].counter;
  });
}

sw_status sw_model_state_info(sw_model* model, uint64_t* step, uint64_t* seed) {
  return sw::guarded([&] {
    require(model, "model");
    if (step) *step = model->model->step();
    if (seed) *seed = model->model->seed();
  });
}

sw_status sw_checkpoint_read(const char* path, sw_checkpoint** out) {
  return sw::guarded([&] {
    require(path, "path");
    require(out, "out");
    auto* ck = new sw_checkpoint{sw::read_checkpoint(path)};
    *out = ck;
  });
}

sw_status sw_checkpoint_info(const sw_checkpoint* ck, uint64_t* step, uint64_t* seed, uint32_t* n_rngs,
                             uint64_t* n_records) {
  return sw::guarded([&] {
    require(ck, "checkpoint");
    if (step) *step = ck->ck.step;
    if (seed) *seed = ck->ck.seed;
    if (n_rngs) *n_rngs = static_cast<uint32_t>(ck->ck.rngs.size());
    if (n_records) *n_records = ck->ck.records.size();
  });
}

sw_status sw_checkpoint_rng(const sw_checkpoint* ck, uint32_t index, const char** name, uint64_t* seed,
                            uint64_t* stream_id, uint64_t* counter) {
  return sw::guarded([&] {
    require(ck, "checkpoint");
    if (index >= ck->ck.rngs.size()) sw::fail(SW_ERR_CONFIG, "checkpoint rng index out of range");
    const sw::CkptRng& r = ck->ck.rngs[index];
    if (name) *name = r.name.c_str();
    if (seed) *seed = r.seed;
    if (stream_id) *stream_id = r.stream_id;
    if (counter) *counter = r.counter;
  });
}

sw_status sw_checkpoint_record(const sw_checkpoint* ck, uint64_t index, const char** name, uint32_t* rank,
                               const int64_t** dims, const float** data, int64_t* numel) {
  return sw::guarded([&] {
    require(ck, "checkpoint");
    if (index >= ck->ck.records.size()) sw::fail(SW_ERR_CONFIG, "checkpoint record index out of range");
    const sw::CkptRecord& r = ck->ck.records[index];
    if (name) *name = r.name.c_str();
    if (rank) *rank = static_cast<uint32_t>(r.shape.size());
    if (dims) *dims = r.shape.data();
    if (data) *data = r.data.data();
    if (numel) *numel = static_cast<int64_t>(r.data.size());
  });
}

sw_status sw_checkpoint_write(const char* path, uint64_t step, uint64_t seed, uint32_t n_rngs,
                              const char* const* rng_names, const uint64_t* rng_seeds, const uint64_t* rng_stream_ids,
                              const uint64_t* rng_counters, uint64_t n_records, const char* const* rec_names,
                              const uint32_t* ranks, const int64_t* const* dims, const float* const* data) {
  return sw::guarded([&] {
    require(path, "path");
    sw::Checkpoint ck;
    ck.step = step;
    ck.seed = seed;
    ck.rngs = rng_list(n_rngs, rng_names, rng_seeds, rng_stream_ids, rng_counters);
    if (n_records > 0) {
      require(rec_names, "rec_names");
      require(ranks, "ranks");
      require(dims, "dims");
      require(data, "data");
    }
    for (uint64_t i = 0; i < n_records; ++i) {
      sw::CkptRecord r;
      r.name = rec_names[i];
      int64_t n = 1;
      for (uint32_t k = 0; k < ranks[i]; ++k) {
        r.shape.push_back(dims[i][k]);
        n *= dims[i][k];
      }
      r.data.assign(data[i], data[i] + n);
      ck.records.push_back(std::move(r));
    }
    sw::write_checkpoint(path, ck);
  });
}

void sw_checkpoint_free(sw_checkpoint* ck) { delete ck; }

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// T5 encoder-decoder extension
// ---------------------------------------------------------------------------------------------
extern "C" {

sw_status sw_t5_create(const sw_model_spec* spec, const sw_plan* plan, sw_mesh* mesh, int batch, int enc_len,
                       int dec_len, sw_t5** out) {
  return sw::guarded([&] {
    require(spec, "spec");
    require(plan, "plan");
    require(mesh, "mesh");
    require(out, "out");
    *out = new sw_t5{new sw::T5Model(spec->spec, plan->plan, mesh->mesh, batch, enc_len, dec_len)};
  });
}

void sw_t5_free(sw_t5* m) {
  if (m != nullptr) {
    delete m->model;
    delete m;
  }
}

sw_status sw_t5_init_params(sw_t5* m, uint64_t seed, const char* stream_name) {
  return sw::guarded([&] {
    require(m, "model");
    require(stream_name, "stream_name");
    m->model->init_params(seed, stream_name);
  });
}

sw_status sw_t5_set_tensor(sw_t5* m, const char* name, int which, const float* full, int64_t numel) {
  return sw::guarded([&] {
    require(m, "model");
    require(name, "name");
    require(full, "full");
    m->model->set_tensor(name, which, full, numel);
  });
}

sw_status sw_t5_get_tensor(sw_t5* m, const char* name, int which, float* full_out, int64_t numel) {
  return sw::guarded([&] {
    require(m, "model");
    require(name, "name");
    require(full_out, "full_out");
    m->model->get_tensor(name, which, full_out, numel);
  });
}

sw_status sw_t5_stage_batch(sw_t5* m, const int32_t* enc_tokens, const int32_t* dec_tokens, const int32_t* targets,
                            const float* weights) {
  return sw::guarded([&] {
    require(m, "model");
    require(enc_tokens, "enc_tokens");
    require(dec_tokens, "dec_tokens");
    require(targets, "targets");
    m->model->stage_batch(enc_tokens, dec_tokens, targets, weights);
  });
}

sw_status sw_t5_forward_backward(sw_t5* m) {
  return sw::guarded([&] {
    require(m, "model");
    m->model->forward_backward();
  });
}

sw_status sw_t5_forward_logits(sw_t5* m, float* logits_out) {
  return sw::guarded([&] {
    require(m, "model");
    require(logits_out, "logits_out");
    m->model->forward_only();
    m->model->logits_to_host(logits_out);
  });
}

sw_status sw_t5_adamw_step(sw_t5* m, const sw_adamw_cfg* cfg) {
  return sw::guarded([&] {
    require(m, "model");
    require(cfg, "cfg");
    m->model->adamw(cfg->lr, cfg->beta1, cfg->beta2, cfg->eps, cfg->weight_decay);
  });
}

sw_status sw_t5_train_step(sw_t5* m, const sw_adamw_cfg* cfg) {
  return sw::guarded([&] {
    require(m, "model");
    require(cfg, "cfg");
    m->model->train_step(cfg->lr, cfg->beta1, cfg->beta2, cfg->eps, cfg->weight_decay);
  });
}

sw_status sw_t5_last_loss(sw_t5* m, double* loss_out) {
  return sw::guarded([&] {
    require(m, "model");
    require(loss_out, "loss_out");
    *loss_out = m->model->last_loss();
  });
}

sw_status sw_t5_stream(sw_t5* m, void** stream_out) {
  return sw::guarded([&] {
    require(m, "model");
    *stream_out = m->model->stream();
  });
}

sw_status sw_t5_set_profiling(sw_t5* m, int enable) {
  return sw::guarded([&] {
    require(m, "model");
    m->model->set_profiling(enable != 0);
  });
}

sw_status sw_t5_read_profile(sw_t5* m, double ms[8], double work[8], int64_t count[8]) {
  return sw::guarded([&] {
    require(m, "model");
    m->model->read_profile(ms, work, count);
  });
}

sw_status sw_t5_launch_count(sw_t5* m, int64_t* out) {
  return sw::guarded([&] {
    require(m, "model");
    *out = m->model->launches();
  });
}

sw_status sw_t5_device_bytes(sw_t5* m, int64_t* out) {
  return sw::guarded([&] {
    require(m, "model");
    *out = m->model->device_bytes();
  });
}

}  // extern "C"
