// C ABI of the mesh and the model program / train state (include/shardweave_b200.h).
#include <cstring>
#include <string>

#include "mesh.h"
#include "model.h"
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
