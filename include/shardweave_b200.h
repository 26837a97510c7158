/*
 * shardweave_b200 — C ABI of the B200-native tensor-parallel transformer step.
 *
 * This is the drop-in boundary for the hot path of the reference ("shardweave", the C++
 * restatement of Redco, arXiv 2310.16355). Every entry point is extern "C", noexcept, takes
 * plain pointers and sizes, and returns an sw_status; sw_last_error() holds the message.
 * Each declaration cites the reference interface it replaces (paths under
 * /root/reference/proj/).
 *
 * Conventions
 *   - Parameter shapes travel as (names[n], ranks[n], dims_flat[sum(ranks)]).
 *   - Kernels are stored [out_features, in_features] exactly as the reference
 *     (graph.hpp:353-375); partitions are "replicated" or "split:<dim>" (partition.hpp:11-39).
 *   - Strings returned as `char**` are malloc'd; release them with sw_free().
 *   - Token ids / labels are int32 (the reference stores them as float and rounds them with
 *     llround, kernels.hpp:21-26).
 *   - `stream` arguments are cudaStream_t passed as void* (NULL = legacy default stream).
 */
#ifndef SHARDWEAVE_B200_H_
#define SHARDWEAVE_B200_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SW_API __attribute__((visibility("default")))
#else
#define SW_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror the reference's exception classes:
 * ShapeError/NonFiniteError (tensor.hpp:37-45), ConfigError/PartitionError/CheckpointError
 * (errors.hpp:10-35), AutodiffError (autodiff.hpp:15-18). */
typedef enum sw_status {
  SW_OK = 0,
  SW_ERR_SHAPE = 1,
  SW_ERR_PARTITION = 2,
  SW_ERR_CONFIG = 3,
  SW_ERR_NONFINITE = 4,
  SW_ERR_CHECKPOINT = 5,
  SW_ERR_AUTODIFF = 6,
  SW_ERR_CUDA = 7,
  SW_ERR_NCCL = 8,
  SW_ERR_INTERNAL = 9
} sw_status;

/* Thread-local message of the last failing call on this thread. */
SW_API const char* sw_last_error(void);
SW_API const char* sw_version(void);
SW_API void sw_free(void* p);

/* ============================================================================================
 * Rule engine (host, bit-exact with the reference)
 * ========================================================================================== */

typedef struct sw_model_spec sw_model_spec;
typedef struct sw_plan sw_plan;

/* Replaces parse_model_spec (model_spec.hpp:30-34, model_spec.cpp:44-119). */
SW_API sw_status sw_model_spec_parse(const char* text, sw_model_spec** out);
/* out[7] = {vocab_size, n_layers, d_model, n_heads, d_ff, max_seq_len, tie_embeddings} */
SW_API sw_status sw_model_spec_dims(const sw_model_spec* spec, int64_t out[7]);
/* Role overrides of the spec as "pattern\trole\n" lines. */
SW_API sw_status sw_model_spec_overrides(const sw_model_spec* spec, char** text_out);
/* Extension keys (not in the reference's spec language): mlp = gelu|swiglu,
 * norm = layernorm|rmsnorm. */
SW_API sw_status sw_model_spec_variant(const sw_model_spec* spec, int* swiglu, int* rmsnorm);
/* Extension: arch = t5 encoder-decoder. out = {is_t5, n_dec_layers, d_kv,
 * rel_buckets, rel_max_distance}. The reference has no encoder-decoder model; the T5 tree is
 * named with its attn / cross_attn / mlp scopes so derive_plan (plan.cpp:39-91) plans it. */
SW_API sw_status sw_model_spec_t5(const sw_model_spec* spec, int64_t out[5]);
/* T5 relative-position bucket ids [tq, tk] (rp = key - query) for a bidirectional (encoder)
 * or causal (decoder) stack. */
SW_API sw_status sw_t5_rel_buckets(int64_t tq, int64_t tk, int bidirectional, int num_buckets,
                                   int max_distance, int32_t* out);
SW_API void sw_model_spec_free(sw_model_spec* spec);

/* Replaces transformer_param_shapes (model.hpp:17-43): "name\td0,d1\n" in tree order. */
SW_API sw_status sw_transformer_param_shapes(const sw_model_spec* spec, char** text_out);

/* Replaces infer_roles (roles.hpp:58-64, roles.cpp:150-189). Output lines
 * "name\trole\tsequence_index\n"; warnings joined by '\n'. */
SW_API sw_status sw_infer_roles(const char* const* names, const int32_t* ranks, const int64_t* dims,
                         size_t n, const char* const* override_patterns,
                         const char* const* override_roles, size_t n_overrides, char** roles_out,
                         char** warnings_out);

/* Replaces derive_plan(ParamTree, n_shards, overrides) (plan.hpp:35-47, plan.cpp:39-91),
 * including role-inference warnings folded in front (plan.hpp:40-47). */
SW_API sw_status sw_plan_derive(const char* const* names, const int32_t* ranks, const int64_t* dims,
                         size_t n, const char* const* override_patterns,
                         const char* const* override_roles, size_t n_overrides, int n_shards,
                         sw_plan** out);
/* Replaces parse_plan (plan.cpp:196-239). */
SW_API sw_status sw_plan_parse(const char* text, int n_shards, sw_plan** out);
/* Replaces serialize_plan (plan.cpp:181-194). */
SW_API sw_status sw_plan_serialize(const sw_plan* plan, char** text_out);
/* Replaces validate_plan (plan.cpp:93-179): violations joined by '\n' (empty = valid). */
SW_API sw_status sw_plan_validate(const sw_plan* plan, const char* const* names, const int32_t* ranks,
                           const int64_t* dims, size_t n, char** violations_out);
SW_API sw_status sw_plan_warnings(const sw_plan* plan, char** text_out);
SW_API sw_status sw_plan_size(const sw_plan* plan, size_t* n_entries, int* n_shards);
/* kind: 0 replicated, 1 split (dim valid). */
SW_API sw_status sw_plan_entry(const sw_plan* plan, size_t i, const char** name, int* kind, int64_t* dim);
SW_API void sw_plan_free(sw_plan* plan);

/* Shard index map (sharded_tensor.hpp:14-36, :52-74): the local shape of `rank` and the
 * [begin, end) range it owns along the split dim (0..size for replicated). */
SW_API sw_status sw_shard_range(const int64_t* global_dims, int32_t rank_of_tensor, int kind,
                         int64_t dim, int n_shards, int shard_rank, int64_t* local_dims_out,
                         int64_t* begin_out, int64_t* end_out);

/* expected_state_elements (train_state.hpp:236-245). */
SW_API sw_status sw_expected_state_elements(const sw_plan* plan, const char* const* names,
                                     const int32_t* ranks, const int64_t* dims, size_t n,
                                     int mp_size, int64_t* out);

/* RngStream(seed, stream_name)[.child(child_index) when >= 0].permutation(n) (rng.hpp:49-65):
 * the Trainer's per-epoch shuffle (pipeline.hpp:383-385). */
SW_API sw_status sw_rng_permutation(uint64_t seed, const char* stream_name, int64_t child_index,
                                    uint64_t n, uint64_t* out);

/* ============================================================================================
 * Mesh and collectives
 * ========================================================================================== */

typedef struct sw_mesh sw_mesh;

/* NCCL unique id (128 bytes) for sw_mesh_create; rank 0 creates it and broadcasts it. */
SW_API sw_status sw_nccl_unique_id(uint8_t out[128]);

/* Replaces build_mesh (mesh.hpp:47-52, mesh.cpp:27-57). device_id = dp_index*mp + mp_index.
 *   world == 1 : every device of the dp x mp mesh lives in this process on `cuda_device`
 *                (collectives are device kernels summing in ascending rank order, like
 *                collectives.hpp:27-52) — the single-GPU emulation of the mesh;
 *   world == dp*mp : one device per process; `rank` is this process's device id and
 *                collectives run on NCCL communicators split per mp group / dp group. */
SW_API sw_status sw_mesh_create(int dp, int mp, int n_hosts, int rank, int world,
                         const uint8_t* nccl_id, int cuda_device, sw_mesh** out);
/* CommReport::to_csv (mesh.cpp:128-138) of everything this mesh communicated. */
SW_API sw_status sw_mesh_comm_report(const sw_mesh* mesh, char** csv_out);
SW_API sw_status sw_mesh_reset_comm_report(sw_mesh* mesh);
SW_API void sw_mesh_free(sw_mesh* mesh);

/* ============================================================================================
 * Model program + train state (spmd_forward_backward / TrainState / adamw_step)
 * ========================================================================================== */

typedef struct sw_model sw_model;

/* AdamWConfig (train_state.hpp:172-178). */
typedef struct sw_adamw_cfg {
  double lr;
  double beta1;
  double beta2;
  double eps;
  double weight_decay;
} sw_adamw_cfg;

/* Lowers transformer_loss(spec, batch, seq_len) (model.hpp:144-152) onto the mesh with the
 * plan: shard materialiser layout (train_state.hpp:50-74), device buffers, kernel schedule.
 * `batch` is the per-replica batch (rows of each dp slice, spmd.hpp:751-769). */
SW_API sw_status sw_model_create(const sw_model_spec* spec, const sw_plan* plan, sw_mesh* mesh,
                          int batch, int seq_len, sw_model** out);
/* The same program for the Predictor path only (cli.cpp:425-447, pipeline.hpp:189-246:
 * predict / generate on restored parameters): bf16 GEMM weight shards, fp32 small parameters
 * and the K/V cache; no gradients, AdamW moments or fp32 master copies of the GEMM weights.
 * forward_logits / last_loss / generate / set_param / get_tensor(which 0) / load_checkpoint
 * (parameters only) work; the training entry points return SW_ERR_CONFIG. */
SW_API sw_status sw_model_create_inference(const sw_model_spec* spec, const sw_plan* plan, sw_mesh* mesh,
                                           int batch, int seq_len, sw_model** out);
SW_API void sw_model_free(sw_model* model);

/* init_transformer_params(spec, RngStream(seed, stream_name)) (model.hpp:49-70), generated
 * on the device from the same counter-based splitmix64 stream (rng.hpp:15-91). */
SW_API sw_status sw_model_init_params(sw_model* model, uint64_t seed, const char* stream_name);
/* Materialise one full host tensor (fp32, row-major) onto this process's shards. */
SW_API sw_status sw_model_set_param(sw_model* model, const char* name, const float* full, int64_t numel);
/* gather (sharded_tensor.hpp:78-98) of replica 0's shards of a parameter / its gradient /
 * its AdamW moments (which: 0 param, 1 grad, 2 adam_m, 3 adam_v) into a full host tensor. */
SW_API sw_status sw_model_get_tensor(sw_model* model, const char* name, int which, float* full_out,
                              int64_t numel);

/* Copies one global batch (dp*batch rows of seq_len) from host memory to the devices.
 * weights may be NULL (all ones). */
SW_API sw_status sw_model_stage_batch(sw_model* model, const int32_t* tokens, const int32_t* targets,
                               const float* weights);
/* spmd_forward_backward for every replica (spmd.hpp:782-814) on the staged batch; gradients
 * are written (accumulate = 0) or added (accumulate = 1) into the grad buffers. */
SW_API sw_status sw_model_forward_backward(sw_model* model, int accumulate);
/* scale_grads (train_state.hpp:146-150). */
SW_API sw_status sw_model_scale_grads(sw_model* model, double factor);
/* dp_sync_grads (train_state.hpp:155-170). */
SW_API sw_status sw_model_dp_sync(sw_model* model);
/* adamw_step (train_state.hpp:183-220); check_finite mirrors its NonFiniteError check. */
SW_API sw_status sw_model_adamw_step(sw_model* model, const sw_adamw_cfg* cfg, int check_finite);
/* One optimizer step of Trainer::fit (pipeline.hpp:388-449) with accumulate_grad_batches=1:
 * forward_backward + dp_sync + adamw. */
SW_API sw_status sw_model_train_step(sw_model* model, const sw_adamw_cfg* cfg);
/* Mean over replicas of the last forward's weighted-mean loss (pipeline.hpp:425-426).
 * Synchronises the device. */
SW_API sw_status sw_model_last_loss(sw_model* model, double* loss_out);
/* Logits [dp*batch, seq_len, vocab] of the staged batch (transformer_logits, model.hpp:76-139). */
SW_API sw_status sw_model_forward_logits(sw_model* model, float* logits_out);
/* Device stream used by this process's first local device (cudaStream_t as void*). */
SW_API sw_status sw_model_stream(sw_model* model, void** stream_out);
/* Number of kernel launches issued by the last forward_backward/adamw/train_step call. */
SW_API sw_status sw_model_launch_count(sw_model* model, int64_t* out);
/* Per-launch device timing with CUDA events on the model stream (categories: 0 GEMM,
 * 1 attention fwd, 2 attention bwd, 3 LayerNorm, 4 cross entropy, 5 AdamW, 6 collectives,
 * 7 other). read_profile returns, per category since the last read: device ms, algorithmic
 * work (FLOPs for 0-2, HBM bytes for 3-5, bus bytes for 6) and launch count. */
SW_API sw_status sw_model_set_profiling(sw_model* model, int enable);
SW_API sw_status sw_model_read_profile(sw_model* model, double ms[8], double work[8],
                                       int64_t count[8]);
/* Bytes of device memory held by this process's model state and activations. */
SW_API sw_status sw_model_device_bytes(sw_model* model, int64_t* out);

/* ==========================================================================================
 * Extension (BASELINE cfg4): T5 encoder-decoder step. The reference has no
 * encoder-decoder; the program is oracle/t5_ref.py's composition of the reference's ops, run
 * under the plan derive_plan (plan.cpp:39-91) gives the T5 tree (arch = t5 spec). dp = 1,
 * tensor parallel over the mesh's mp axis, replicated lm_head.
 * ========================================================================================== */
typedef struct sw_t5 sw_t5;
/* batch rows of enc_len encoder tokens and dec_len decoder tokens (<= max_seq_len). */
SW_API sw_status sw_t5_create(const sw_model_spec* spec, const sw_plan* plan, sw_mesh* mesh, int batch,
                              int enc_len, int dec_len, sw_t5** out);
SW_API void sw_t5_free(sw_t5* model);
/* init_transformer_params' rules (model.hpp:49-70) over the T5 tree, same device stream. */
SW_API sw_status sw_t5_init_params(sw_t5* model, uint64_t seed, const char* stream_name);
/* which: 0 param (+ bf16 shadow), 2 adam_m, 3 adam_v (set); 0..3 incl. 1 grad (get). */
SW_API sw_status sw_t5_set_tensor(sw_t5* model, const char* name, int which, const float* full,
                                  int64_t numel);
SW_API sw_status sw_t5_get_tensor(sw_t5* model, const char* name, int which, float* full_out,
                                  int64_t numel);
/* enc_tokens [batch, enc_len]; dec_tokens / targets / weights [batch, dec_len]; weights may be
 * NULL (all ones). */
SW_API sw_status sw_t5_stage_batch(sw_t5* model, const int32_t* enc_tokens, const int32_t* dec_tokens,
                                   const int32_t* targets, const float* weights);
/* Weighted-mean cross entropy and every parameter gradient (written, not accumulated). */
SW_API sw_status sw_t5_forward_backward(sw_t5* model);
/* Decoder logits [batch * dec_len, vocab] of the staged batch. */
SW_API sw_status sw_t5_forward_logits(sw_t5* model, float* logits_out);
SW_API sw_status sw_t5_adamw_step(sw_t5* model, const sw_adamw_cfg* cfg);
SW_API sw_status sw_t5_train_step(sw_t5* model, const sw_adamw_cfg* cfg);
SW_API sw_status sw_t5_last_loss(sw_t5* model, double* loss_out);
SW_API sw_status sw_t5_stream(sw_t5* model, void** stream_out);
SW_API sw_status sw_t5_set_profiling(sw_t5* model, int enable);
SW_API sw_status sw_t5_read_profile(sw_t5* model, double ms[8], double work[8], int64_t count[8]);
SW_API sw_status sw_t5_launch_count(sw_t5* model, int64_t* out);
SW_API sw_status sw_t5_device_bytes(sw_t5* model, int64_t* out);

/* Greedy next-token generation: the Predictor loop of cli.cpp:425-447 (window of the last
 * seq_len tokens, argmax at the newest position, kernels.hpp:515-527 first-maximum rule) for
 * `batch` rows of P prompt tokens each, n_new tokens per row -> out [batch, n_new]. While the
 * context fits the window each step runs one position through a KV cache; after that the window
 * slides and is re-run with positions 0..seq_len-1, as the reference does. Replica 0's state. */
SW_API sw_status sw_model_generate(sw_model* model, const int32_t* prompts, int P, int n_new, int32_t* out);

/* ============================================================================================
 * SWCK train-state snapshots (checkpoint.hpp:18-28 format, byte-compatible with the reference)
 * ========================================================================================== */

/* save_checkpoint (checkpoint.hpp:193-220): the optimizer step, the state seed (the init seed),
 * the given named RNG streams, then replica 0's gathered params / adam_m / adam_v in tree order
 * (model.hpp:17-43). Under NCCL every rank calls it (the gathers are collective over the mp
 * group) and world rank 0 writes the file. */
SW_API sw_status sw_model_save_checkpoint(sw_model* model, const char* path, uint32_t n_rngs,
                                          const char* const* rng_names, const uint64_t* rng_seeds,
                                          const uint64_t* rng_stream_ids, const uint64_t* rng_counters);
/* load_checkpoint (checkpoint.hpp:233-298): validates the file (SW_ERR_CHECKPOINT with the
 * reference's message and "(at byte offset N)"), re-cuts every tensor onto this model's plan and
 * mesh, and restores the optimizer step. *n_rngs_out (may be NULL) receives the number of RNG
 * streams stored; read them with sw_model_checkpoint_rng. */
SW_API sw_status sw_model_load_checkpoint(sw_model* model, const char* path, uint32_t* n_rngs_out);
SW_API sw_status sw_model_checkpoint_rng(sw_model* model, uint32_t index, char* name, uint64_t name_cap,
                                         uint64_t* seed, uint64_t* stream_id, uint64_t* counter);
/* TrainState step / seed (train_state.hpp:24-27). */
SW_API sw_status sw_model_state_info(sw_model* model, uint64_t* step, uint64_t* seed);

/* Host-only SWCK codec (no device): parse or write a snapshot file. Records are the
 * params/x, adam_m/x, adam_v/x triples in file order; only f32 payloads (the executor's
 * Scalar) are accepted, like load_checkpoint<float>. */
typedef struct sw_checkpoint sw_checkpoint;
SW_API sw_status sw_checkpoint_read(const char* path, sw_checkpoint** out);
SW_API sw_status sw_checkpoint_info(const sw_checkpoint* ck, uint64_t* step, uint64_t* seed, uint32_t* n_rngs,
                                    uint64_t* n_records);
SW_API sw_status sw_checkpoint_rng(const sw_checkpoint* ck, uint32_t index, const char** name, uint64_t* seed,
                                   uint64_t* stream_id, uint64_t* counter);
SW_API sw_status sw_checkpoint_record(const sw_checkpoint* ck, uint64_t index, const char** name,
                                      uint32_t* rank, const int64_t** dims, const float** data,
                                      int64_t* numel);
SW_API sw_status sw_checkpoint_write(const char* path, uint64_t step, uint64_t seed, uint32_t n_rngs,
                                     const char* const* rng_names, const uint64_t* rng_seeds,
                                     const uint64_t* rng_stream_ids, const uint64_t* rng_counters,
                                     uint64_t n_records, const char* const* rec_names, const uint32_t* ranks,
                                     const int64_t* const* dims, const float* const* data);
SW_API void sw_checkpoint_free(sw_checkpoint* ck);

/* ============================================================================================
 * Kernel-level entry points (device pointers). Used by the parity tests and the roofline
 * measurements; each is one launch on `stream`.
 * ========================================================================================== */

/* C[M,N] = sum_k A[m,k] B[n,k] — bf16 in, fp32 accumulate (tcgen05). a_mn_major / b_mn_major
 * select the operand layouts; epi: 0 bf16, 1 f32 (+accumulate), 2 bias+gelu (C=pre, C2=act),
 * 3 residual f32 (C = aux + acc + bias), 4 gelu-backward (C = acc * gelu'(aux)), 8 attention
 * output gradient with the backward's row statistic: C = bf16(acc) and, with C2 = fp32 delta
 * [M / ldc2][N / 128][ldc2] and ldc2 = sequence length, delta[b][h][t] = sum over the 128 columns
 * of head h of C[b*ldc2 + t, c] * aux[b*ldc2 + t, c] (aux = bf16 attention output O). */
SW_API sw_status sw_k_gemm_bf16(int M, int N, int K, const void* A, int64_t lda, int a_mn_major,
                         const void* B, int64_t ldb, int b_mn_major, int epi, void* C, int64_t ldc,
                         void* C2, int64_t ldc2, const float* bias, const void* aux,
                         int64_t ld_aux, float alpha, int accumulate, void* stream);

/* Causal attention over head-sharded activations (graph.hpp:650-661 + model.hpp:100-106):
 * qkv [B*T, 3*Hl*hd] bf16 (q | k | v), o [B*T, Hl*hd] bf16, lse [B, Hl, T] fp32. */
/* One cached decode step of attention (the Predictor's KV-cached next token):
 * qkv_new [B, 3*Hl*hd] bf16 is the step's q | k | v row per sequence; cache [B*T, 3*Hl*hd] bf16
 * holds keys/values 0..p-1 (the layer's qkv activations); out [B, Hl*hd] bf16. split != 0: the
 * split-key kernel, which also writes the new k | v into cache row p (part: B*Hl*16*(hd+2)
 * floats, ticket: B*Hl zero-initialised uints); split == 0: kv scatter + the one-CTA-per-head
 * kernel. */
SW_API sw_status sw_k_decode_attention(const void* qkv_new, void* cache, void* out, int B, int T, int p, int Hl,
                                       int hd, int split, float* part, unsigned int* ticket, void* stream);
SW_API sw_status sw_k_attention_fwd(const void* qkv, void* o, float* lse, int B, int T, int Hl,
                                    int hd, void* stream);
/* dqkv [B*T, 3*Hl*hd] bf16; scratch fp32 of sw_k_attention_bwd_scratch(B, T, Hl, hd) elements. */
SW_API sw_status sw_k_attention_bwd(const void* qkv, const void* o, const float* lse,
                                    const void* dout, void* dqkv, float* scratch, int B, int T,
                                    int Hl, int hd, void* stream);
/* fp32 elements of sw_k_attention_bwd's scratch (delta, and the fp32 dQ accumulator or, for
 * head_dim 128 with T % 128 == 0, the dS^T tiles of the query-block dQ kernel). */
SW_API long long sw_k_attention_bwd_scratch(int B, int T, int Hl, int hd);
/* Debug/profiling only: 4096 clock64 stamps of the attention-backward CTA named by the
 * SW_ATTN_TRACE_CTA environment variable (slot map in tools/attn_trace.py). */
SW_API sw_status sw_k_attention_trace(unsigned long long* out);
/* Debug/profiling only: 1024 per-tile phase stamps of the CTA-pair GEMM CTA named by
 * SW_GEMM_TRACE_CTA (slot map in tools/gemm_trace.py). */
SW_API sw_status sw_k_gemm_trace(unsigned long long* out);
/* LayerNorm (kernels.hpp:184-271): y bf16, mean/rstd fp32 [M]. */
SW_API sw_status sw_k_layernorm_fwd(const float* x, const float* scale, const float* bias, void* y,
                                    float* mean, float* rstd, int64_t M, int d, float eps,
                                    void* stream);
SW_API sw_status sw_k_layernorm_bwd(const float* x, const float* mean, const float* rstd,
                                    const float* scale, const float* dy, float* g_io, void* g_bf16,
                                    float* dscale, float* dbias, int64_t M, int d, int accumulate,
                                    void* stream);
/* Fused softmax cross entropy fwd+bwd over bf16 logits [M, ld] (kernels.hpp:327-363). */
/* RMSNorm (extension): y = x / sqrt(mean(x^2) + eps) * scale (bf16 out), rstd saved;
 * backward dx = rstd*(g - xhat*mean(g*xhat)), g = dy*scale, with g_io / g_bf16 / dscale as in
 * sw_k_layernorm_bwd (dscale accumulated). */
SW_API sw_status sw_k_rmsnorm_fwd(const float* x, const float* scale, void* y, float* rstd, int64_t M, int d,
                                  float eps, void* stream);
SW_API sw_status sw_k_rmsnorm_bwd(const float* x, const float* rstd, const float* scale, const float* dy,
                                  float* g_io, void* g_bf16, float* dscale, int64_t M, int d, int accumulate,
                                  void* stream);
SW_API sw_status sw_k_xent(void* logits, int64_t ld, int64_t M, int V, const int32_t* targets,
                           const float* weights, const float* wsum, float* wloss, int write_grad,
                           void* stream);
/* AdamW over a flat shard (train_state.hpp:211-216), bf16 shadow refresh. */
SW_API sw_status sw_k_adamw(float* p, float* m, float* v, const float* g, void* shadow, int64_t n,
                            float lr, float b1, float b2, float eps, float wd, float c1, float c2,
                            void* stream);

/* SwiGLU MLP (extension): with W_gu = [gate; up] [2N, K] (K-major), h[M,N] =
 * silu(A W_gate^T) * (A W_up^T) and pre[M, 2N] = bf16(A W_gate^T) | bf16(A W_up^T), one GEMM.
 * The backward fuses the SwiGLU derivative into the down-projection dgrad: acc = dY . W_down
 * [M, N]; dpre[M, 2N] = acc*u*silu'(g) | acc*silu(g) from pre. All bf16. */
SW_API sw_status sw_k_gemm_bf16_swiglu(int M, int N, int K, const void* A, int64_t lda, const void* W_gu, int64_t ldw,
                                       void* h, int64_t ldh, void* pre, int64_t ldpre, void* stream);
SW_API sw_status sw_k_gemm_bf16_swiglu_bwd(int M, int N, int K, const void* A, int64_t lda, int a_mn_major,
                                           const void* B, int64_t ldb, int b_mn_major, const void* pre,
                                           int64_t ldpre, void* dpre, int64_t lddpre, void* stream);

/* Optimizer in the backward: the weight-gradient GEMM G[M,N] = A^T-or-A . B (same operand
 * conventions as sw_k_gemm_bf16) whose epilogue applies the AdamW update of sw_k_adamw
 * (train_state.hpp:214-216) to p/m/v [M, ld] in place and refreshes the bf16 shadow; G is never
 * stored. *nonfinite_flag is OR-ed with 1 when any gradient element is non-finite. */
SW_API sw_status sw_k_gemm_bf16_adamw(int M, int N, int K, const void* A, int64_t lda, int a_mn_major,
                                      const void* B, int64_t ldb, int b_mn_major, float* p, float* m, float* v,
                                      void* shadow, int64_t ld, int* nonfinite_flag, float lr, float b1, float b2,
                                      float eps, float wd, float c1, float c2, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SHARDWEAVE_B200_H_ */
