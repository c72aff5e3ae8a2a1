/*
 * mugv_b200 — C ABI of the B200-native MUG-V DiT-block hot path.
 *
 * Drop-in boundary for the reference's C++ value API (proj/include/mugv/dit.hpp,
 * proj/include/mugv/flowtrain.hpp).  Plain C types only: pointers, sizes, POD
 * structs.  Every entry point is re-entrant per context, never throws, and
 * returns an mgv_status; mgv_last_error(ctx) holds the message.  Host buffers
 * are fp64 like the reference's Tensor (proj/include/mugv/tensor.hpp:11);
 * device compute is bf16 tensor-core (MGV_PREC_BF16) or IEEE fp32 (MGV_PREC_FP32,
 * <= 1e-4 relative to the fp64 reference).
 *
 * Reference interface each entry point replaces:
 *   mgv_params_upload        ParameterSet handed to every call      proj/include/mugv/params.hpp:28-52
 *                            (weights are cached on device; re-upload when they change)
 *   mgv_params_init          dit::init_dit_params (+ the tests' gate opening)  proj/src/dit.cpp:143-183
 *   mgv_predict_velocity     dit::predict_velocity                  proj/include/mugv/dit.hpp:104-106
 *   mgv_velocity_graph       dit::velocity_rows_graph (tape node + backward closure)  proj/include/mugv/dit.hpp:124-127
 *   mgv_dit_forward          dit::dit_forward                       proj/include/mugv/dit.hpp:94-95
 *                            (dit_forward_batch, dit.hpp:98-100, is a loop of this call)
 *   mgv_flow_step            flow::FlowTrainer::step: loss, backward, proj/include/mugv/flowtrain.hpp:134-151
 *                            grad_norm, AdamW (mgv_ctx_set_adamw)   proj/src/flowtrain.cpp:257-289
 *   mgv_flow_loss            flow::flow_loss                        proj/include/mugv/flowtrain.hpp:26
 *   mgv_latent_rows          dit::latent_rows                       proj/include/mugv/dit.hpp:58
 *   mgv_patchify             dit::patchify                          proj/include/mugv/dit.hpp:86-87
 *   mgv_unpatchify           dit::unpatchify                        proj/include/mugv/dit.hpp:89-90
 *   mgv_global_embed         dit::global_embed                      proj/include/mugv/dit.hpp:83-84
 *   mgv_fused_modulate       SPEC fused_modulate (no code in proj/)
 *   mgv_apply_rope3d         Tape::rope3d / SPEC apply_rope3d        proj/src/autodiff.cpp:849-898
 *   mgv_tokenize             dit::tokenize                          proj/src/dit.cpp:193-211
 *   mgv_text_embed           dit::text_embed                        proj/include/mugv/dit.hpp:63-72, dit.cpp:213-234
 *   mgv_rows_to_grid         dit::rows_to_grid                      proj/include/mugv/dit.hpp:62
 *   mgv_ckpt_load / _read    mugv::load_checkpoint                  proj/include/mugv/params.hpp:60, params.cpp:128-225
 *   mgv_ckpt_save            mugv::save_checkpoint                  proj/include/mugv/params.hpp:59, params.cpp:92-126
 *   mgv_params_upload_ckpt   load_checkpoint -> ParameterSet handed to the hot path (device upload, no fp64 trip)
 *   mgv_params_save          save_checkpoint of the trained dit.* parameters (device fp32 masters)
 *   mgv_flow_errors          post::flow_error (forward only)        proj/include/mugv/posttrain.hpp:72-75
 *   mgv_flow_step_weighted   the tape of post_loss_graph: sum_k w_k dl_k, grad_norm, AdamW
 *   mgv_post_*               post::PostTrainState / post_train_step / post_loss_graph / dpo_loss / kto_loss
 *                                                                   proj/include/mugv/posttrain.hpp:83-154
 */
#ifndef MUGV_B200_H
#define MUGV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mgv_ctx mgv_ctx;

/* mirrors the reference's exception taxonomy (proj/include/mugv/errors.hpp:13-30) + device errors */
typedef enum {
    MGV_OK = 0,
    MGV_ERR_DIMENSION = 1, /* DimensionError */
    MGV_ERR_CONFIG = 2,    /* ConfigError */
    MGV_ERR_INPUT = 3,     /* InputError */
    MGV_ERR_NUMERIC = 4,   /* NumericError */
    MGV_ERR_CUDA = 5,
    MGV_ERR_NCCL = 6,
    MGV_ERR_INTERNAL = 7,
    MGV_ERR_CHECKPOINT = 8, /* CheckpointError; kind from mgv_ckpt_last_error_kind() */
    MGV_ERR_SCHEDULING = 9  /* SchedulingError (post-training interleave plan) */
} mgv_status;

typedef enum { MGV_PREC_FP32 = 0, MGV_PREC_BF16 = 1 } mgv_precision;

/* dit::DitConfig (proj/include/mugv/dit.hpp:13-26) */
typedef struct {
    int64_t depth, hidden, heads, text_dim, c_z;
    int32_t rope_split[3];
    int64_t text_vocab, text_max_len;
} mgv_dit_cfg;

/* One flow::FlowSample (flowtrain.hpp:111-117), rows already patchified (N = dims[0]*dims[1]*dims[2]).
 * conditioned: N flags (NULL = no conditioning), any unit-aligned mask (flowtrain.cpp:61-100);
 * condition_latents: N x 4c_z rows, read at conditioned rows (first_frame_mask passes clean_rows); NULL with a
 * conditioned token is MGV_ERR_INPUT as in validate_mask (flowtrain.cpp:77-80).  mgv_flow_step_device takes
 * device pointers here, the mask unvalidated, and NULL condition_latents = clean_rows. */
typedef struct {
    int64_t dims[3];
    const int32_t* coords; /* N x 3 (t, py, px) */
    const double* clean_rows;
    const double* noise;
    double t;
    const uint8_t* conditioned;
    const double* condition_latents;
} mgv_flow_sample;

/* One flow-error evaluation of post-training (posttrain.hpp:15-21 SampleRecord at its SharedDraw :66-69):
 * s.clean_rows = the record's latent rows, s.noise / s.t = the shared draw, s.conditioned /
 * s.condition_latents = the record's ConditionMask (first-frame masks), plus the record's own text and fps. */
typedef struct {
    mgv_flow_sample s;
    const double* text; /* L x text_dim */
    int64_t L;
    double fps;
} mgv_eval_sample;

mgv_status mgv_ctx_create(int device, int precision, mgv_ctx** out);
void mgv_ctx_destroy(mgv_ctx* ctx);
const char* mgv_last_error(mgv_ctx* ctx);
/* 0 = default; else a cudaStream_t the context launches on */
mgv_status mgv_ctx_set_stream(mgv_ctx* ctx, void* stream);

/* Data parallel: rank r of `world` over NCCL; `nccl_id` is the 128-byte ncclUniqueId from rank 0.
 * mgv_flow_step then all-reduces gradients (sum) and scales the loss by 1/global_batch.  world 1 with an id
 * builds a one-rank communicator (the all-reduce path runs, as an identity).  nccl_id NULL with world > 1: no
 * communicator -- the step returns this rank's share (loss and gradients scaled by 1/global_batch, unreduced;
 * their sum over the ranks is the global step; leave AdamW off in this mode). */
mgv_status mgv_nccl_unique_id(uint8_t out[128]);
mgv_status mgv_ctx_set_dp(mgv_ctx* ctx, int rank, int world, const uint8_t nccl_id[128]);
/* Tensor parallel (Megatron head/column split); must precede mgv_params_upload.
 * nccl_id != NULL: this context is TP rank `rank` of `size` over NCCL: it stores only its blocks of the
 * sharded parameters and H/size-wide activations; one exchange per residual branch in forward and backward
 * (NVLink peer memory fused into the row-parallel GEMM epilogue, or NCCL); no gradient all-reduce; the
 * gradient norm is summed over the group; parameter / gradient downloads all-gather the blocks (collective).
 * nccl_id == NULL: all `size` ranks are emulated in this context (every slot held, partial sums accumulated
 * in place of the exchange) -- the single-GPU check of the sharded path.  `size` must divide heads.
 * Combinable with mgv_ctx_set_dp (2-D: the DP communicator joins the ranks holding the same TP rank; the DP
 * gradient all-reduce then runs once after the backward instead of in per-block buckets). */
mgv_status mgv_ctx_set_tp(mgv_ctx* ctx, int size, int rank, const uint8_t* nccl_id);

/* flow::forward_sample_rows (direction -1: Euler t 1 -> 0, x <- x - dt v) and flow::reverse_sample_rows
 * (direction +1: t 0 -> 1, x <- x + dt v), flowtrain.cpp:135-172 / flowtrain.hpp:66-76, with the model
 * velocity of flow::model_velocity (:102-107): x_start (N x 4c_z) on the grid dims/coords, `steps` >= 1
 * steps run on device, conditioned rows (mask `conditioned`, N bytes, may be NULL) re-imposed from
 * condition_latents (N x 4c_z) before and after every step.  Errors as the reference (InputError for
 * steps < 1 or a unit-misaligned mask, DimensionError for shape mismatches). */
mgv_status mgv_sample_rows(mgv_ctx* ctx, const double* x_start, int64_t N, const int32_t* coords,
                           const int64_t dims[3], const double* text, int64_t L, const uint8_t* conditioned,
                           const double* condition_latents, int64_t steps, int direction, double fps, double* out);

/* AdamW (replaces mugv::AdamW, optim.hpp:12-29 / optim.cpp:7-24): when lr > 0, every mgv_flow_step /
 * mgv_flow_step_device ends with AdamW::update over all dit.* parameters on device (fp32 masters, m and v
 * resident, bf16 operand copies refreshed) -- the full FlowTrainer::step (flowtrain.cpp:257-282).  The
 * update is skipped when the loss is not finite (the step then fails with MGV_ERR_NUMERIC, as the
 * reference throws before updating).  Uploading parameters resets the optimizer state. */
mgv_status mgv_ctx_set_adamw(mgv_ctx* ctx, double lr, double beta1, double beta2, double eps, double weight_decay);
int64_t mgv_adamw_steps(mgv_ctx* ctx); /* AdamW::step_count (optim.hpp:24) */
/* Read parameter i (sorted-name order, mgv_param_name) back in the reference layout, fp64. */
mgv_status mgv_param_download(mgv_ctx* ctx, int64_t i, double* out);

/* dit::init_dit_params (dit.cpp:143-183) with mugv::Rng(seed), uploaded (bit-identical to the reference's weights);
 * gate_seed != 0 then redraws dit.mod.{w,b} / dit.final.w (std gate_std) and dit.final.b (gate_b_std) from
 * Rng(gate_seed), the tests' open_gates (test_dit.cpp:35-41). */
mgv_status mgv_params_init(mgv_ctx* ctx, const mgv_dit_cfg* cfg, uint64_t seed, uint64_t gate_seed, double gate_std,
                           double gate_b_std);
/* Seeded synthetic inputs with the reference's streams: Rng(seed).uniform_tensor (rng.hpp:60-64), and
 * flow::make_batch (flowtrain.cpp:231-250) for one sample: noise, t, and the first-frame mask draw. */
mgv_status mgv_rng_uniform_fill(uint64_t seed, int64_t n, double lo, double hi, double* out);
mgv_status mgv_make_flow_sample(uint64_t seed, int64_t N, int64_t D, double mask_prob, double* noise, double* t,
                                int* conditioned);
/* Varlen packing (BASELINE configs[4]): on != 0 runs every multi-sample flow step as ONE packed sequence of
 * 256-row-aligned segments with block-diagonal attention, per-sample timesteps in the modulation table and
 * per-sample masked-mean losses (flowtrain.cpp:263-273): each sample's forward is bit-identical to running it
 * alone; gradients equal the per-sample sum up to summation order.  Default off (samples run one by one). */
mgv_status mgv_ctx_set_varlen(mgv_ctx* ctx, int on);
/* Per-block activation recompute for training steps (deep stacks at 57,600 tokens): on != 0
 * keeps only every block's input residual rows; the backward re-runs each block's forward (same kernels, same
 * inputs: bit-identical results) before differentiating it.  One extra block forward per block, ~1/depth of the
 * activation memory.  Default off. */
mgv_status mgv_ctx_set_recompute(mgv_ctx* ctx, int on);
/* Memory per rank, out = {parameters (fp32 masters + bf16 operand copies), gradients, AdamW moments, step
 * workspace (saved activations + scratch), TP exchange arena} in bytes.  mgv_plan_rank_bytes plans a step of
 * N tokens (text length L, n_u unique timesteps) for TP degree tp without a device, with the runtime's own
 * layout code (one real TP rank: its parameter blocks and H/P-wide activations); train: 0 forward, 1 training step,
 * 3 training step with per-block recompute (mgv_ctx_set_recompute); mgv_ctx_memory reports what a context holds
 * now (emulated TP ranks hold all P slots). */
mgv_status mgv_plan_rank_bytes(const mgv_dit_cfg* cfg, int precision, int tp, int64_t N, int64_t L, int64_t n_u,
                               int train, int64_t out[5]);
mgv_status mgv_ctx_memory(mgv_ctx* ctx, int64_t out[5]);
/* Upload (or replace) the dit.* ParameterSet.  names/data/numel are n parallel arrays (any order). */
mgv_status mgv_params_upload(mgv_ctx* ctx, const mgv_dit_cfg* cfg, int64_t n, const char* const* names,
                             const double* const* data, const int64_t* numel);
int64_t mgv_param_count(mgv_ctx* ctx);
const char* mgv_param_name(mgv_ctx* ctx, int64_t i); /* sorted-name order = gradient order */
int64_t mgv_param_numel(mgv_ctx* ctx, int64_t i);

/* dit::predict_velocity: rows (N x 4c_z), coords (N x 3), dims (U, H', W'), text (L x text_dim),
 * timesteps (N), fps -> out (N x 4c_z). */
mgv_status mgv_predict_velocity(mgv_ctx* ctx, const double* rows, int64_t N, const int32_t* coords,
                                const int64_t dims[3], const double* text, int64_t L, const double* timesteps,
                                double fps, double* out);

/* The tape-level builder dit::velocity_rows_graph (dit.hpp:124-127, dit.cpp:320-334) as ONE device node, for the
 * TapeOps seam (autodiff.hpp:130-134).  Forward: velocity (N x 4c_z) and, when taps != NULL, the reference's taps
 * in order (depth + 3 pointers, each may be NULL): patch embedding (N x hidden), each block's residual output
 * (N x hidden) x depth, the final normed projection (N x hidden), the velocity rows (N x 4c_z).  Backward (the
 * node's closure): dV != NULL gives the vector-Jacobian product, gradients of sum(dV * velocity) w.r.t. every
 * dit.* parameter written to grads_out (sorted-name order, mgv_param_name; entries may be NULL).  rows and text
 * are constants of the graph, as in every reference caller (flowtrain.cpp:268, posttrain.cpp:132,284,
 * expansion.cpp:267-272). */
mgv_status mgv_velocity_graph(mgv_ctx* ctx, const double* rows, int64_t N, const int32_t* coords,
                              const int64_t dims[3], const double* text, int64_t L, const double* timesteps,
                              double fps, double* velocity, double* const* taps, const double* dV,
                              double* const* grads_out);
/* dit::dit_forward: tokens (N x hidden) -> out (N x hidden). */
mgv_status mgv_dit_forward(mgv_ctx* ctx, const double* tokens, int64_t N, const int32_t* coords,
                           const int64_t dims[3], const double* text, int64_t L, const double* timesteps, double fps,
                           double* out);

/* dit::tokenize: FNV-1a 64 ids of the whitespace-separated words modulo vocab; returns the word count (ids holds
 * the first min(count, cap)), -1 on bad arguments.  Host-only. */
int64_t mgv_tokenize(const char* prompt, int64_t vocab, int64_t* ids, int64_t cap);
/* dit::text_embed: truncate to max_len ids (*truncated = 1 when cut), look up rows of embed_table (vocab x text_dim;
 * the "text.embed" parameter, or null_row "text.null" when empty), RMS-normalise each row on the device in the
 * reference's fp64 order (bit-identical).  out: max(1, min(n, max_len)) x text_dim.  InputError for ids outside
 * the vocabulary. */
mgv_status mgv_text_embed(mgv_ctx* ctx, const int64_t* ids, int64_t n, const double* embed_table, int64_t vocab,
                          const double* null_row, int64_t text_dim, int64_t max_len, double* out, int* truncated);
/* dit::patchify: (U, h, w, C) latent grid -> tokens (N x hidden) = latent_rows(grid) W_patch^T + b_patch, and
 * the N x 3 coords.  DimensionError for odd h / w or C != c_z (dit.cpp:336-345). */
mgv_status mgv_patchify(mgv_ctx* ctx, const double* grid, int64_t U, int64_t h, int64_t w, int64_t C, double* tokens,
                        int32_t* coords);
/* dit::unpatchify: tokens (N x hidden) on coords of a (U, H', W') grid -> (U, 2H', 2W', c_z) grid of the output head
 * W_out tokens + b_out (dit.cpp:347-359). */
mgv_status mgv_unpatchify(mgv_ctx* ctx, const double* tokens, int64_t N, const int32_t* coords, const int64_t dims[3],
                          double* grid);
/* dit::global_embed: g (N x hidden) = gmlp(sinusoid(1000 tau)) + gmlp(sinusoid(fps)) per token, and (if not NULL)
 * block_scales (depth x hidden) = the per-block gscale parameters (dit.cpp:257-265).  InputError for tau outside
 * [0, 1]. */
mgv_status mgv_global_embed(mgv_ctx* ctx, const double* timesteps, int64_t N, double fps, double* g,
                            double* block_scales);

/* ---- SPEC-only operators of the path (no code in proj/) ----
 * mgv_fused_modulate: SPEC.md:616-624  out = residual + ((x + bias) * (1 + scale) + shift) over a rows x cols
 *   fp64 buffer, bias / scale / shift with 1 (scalar), cols (per channel) or rows*cols elements, else
 *   MGV_ERR_DIMENSION; one device pass, bit-identical to the composed three-step reference (no contraction).
 * mgv_dev_fused_modulate_f32: the same operator on DEVICE fp32 buffers (per-channel vectors, cols % 4 == 0,
 *   16-byte aligned), on the context stream, asynchronous; one read of x / residual, one write of out.
 * mgv_apply_rope3d: SPEC.md:168-176, Tape::rope3d forward (autodiff.cpp:849-898): x is N x heads*hd fp64 with
 *   hd = split[0] + split[1] + split[2], coords N x 3 (t, h, w); odd split -> MGV_ERR_CONFIG.  inverse != 0
 *   applies the inverse rotation (the backward's rope_apply_vec(..., -1)).  Bit-identical to the reference. */
mgv_status mgv_fused_modulate(mgv_ctx* ctx, const double* x, const double* bias, int64_t bias_n, const double* scale,
                              int64_t scale_n, const double* shift, int64_t shift_n, const double* residual,
                              int64_t rows, int64_t cols, double* out);
mgv_status mgv_dev_fused_modulate_f32(mgv_ctx* ctx, const float* x, const float* bias, const float* scale,
                                      const float* shift, const float* residual, int64_t rows, int64_t cols,
                                      float* out);
mgv_status mgv_apply_rope3d(mgv_ctx* ctx, const double* x, int64_t N, int64_t heads, const int64_t split[3],
                            const int32_t* coords, double base, int inverse, double* out);

/* FlowTrainer::step forward + backward over n local samples (global_batch = n * world).
 * loss: mean of per-sample masked flow losses; grad_norm: sqrt of the sum of squared gradient entries;
 * grads_out: NULL, or mgv_param_count pointers (sorted-name order, NULL entries skipped) receiving fp64 grads.
 * velocity_out: NULL or n pointers receiving each sample's V rows. */
mgv_status mgv_flow_step(mgv_ctx* ctx, int64_t n, const mgv_flow_sample* samples, const double* text, int64_t L,
                         double fps, double* loss, double* grad_norm, double* const* grads_out,
                         double* const* velocity_out);

/* flow::flow_loss on host-resident rows (N x D) with a per-row mask. */
mgv_status mgv_flow_loss(mgv_ctx* ctx, const double* pred, const double* target, const uint8_t* mask, int64_t N,
                         int64_t D, double* loss);

/* dit::latent_rows / rows_to_grid (bit-exact 2x2 patch index math on device). */
mgv_status mgv_latent_rows(mgv_ctx* ctx, const double* grid, int64_t U, int64_t h, int64_t w, int64_t C,
                           double* rows, int32_t* coords);
mgv_status mgv_rows_to_grid(mgv_ctx* ctx, const double* rows, const int32_t* coords, int64_t N, const int64_t dims[3],
                            int64_t C, double* grid);

/* mgv_flow_step with DEVICE-resident sample/text buffers (same struct, device pointers): the
 * benchmark's inputs-already-in-HBM figure.  No gradients or velocities are read back. */
mgv_status mgv_flow_step_device(mgv_ctx* ctx, int64_t n, const mgv_flow_sample* samples, const double* text_dev,
                                int64_t L, double fps, double* loss, double* grad_norm);

/* Timing / introspection for the benchmark: device time (ms) of the last mgv_flow_step's compute,
 * and the number of kernel launches it issued. */
double mgv_last_step_ms(mgv_ctx* ctx);
int64_t mgv_last_step_launches(mgv_ctx* ctx);
/* Per-phase CUDA-event timing ("attn_fwd", "attn_bwd", "blocks_fwd", "gemm" = every bf16 GEMM launch, ...),
 * accumulated over steps.  mgv_prof_entry_work: the phase's algorithmic FLOPs (2 M N K summed; "gemm" only). */
mgv_status mgv_prof_enable(mgv_ctx* ctx, int on);
int64_t mgv_prof_count(mgv_ctx* ctx);
const char* mgv_prof_entry(mgv_ctx* ctx, int64_t i, double* ms, int64_t* launches);
double mgv_prof_entry_work(mgv_ctx* ctx, int64_t i);

/* ---- MUGVCKPT checkpoint container (proj/include/mugv/params.hpp:54-61, proj/src/params.cpp:92-225) ----
 * Host-only (no device needed).  The writer emits the same bytes as mugv::save_checkpoint for the same
 * ParameterSet; the reader applies the reference's validation with its CheckpointError kinds
 * (errors.hpp:43): a failing call returns MGV_ERR_CHECKPOINT and sets the calling thread's
 * mgv_ckpt_last_error() / mgv_ckpt_last_error_kind().  Entries are in sorted-name order. */
typedef struct mgv_ckpt mgv_ckpt;
typedef enum { MGV_CKPT_F32 = 0, MGV_CKPT_F64 = 1 } mgv_ckpt_dtype_t; /* Dtype (params.hpp:14) */
typedef enum {
    MGV_CKPT_BAD_MAGIC = 0,
    MGV_CKPT_TRUNCATED = 1,
    MGV_CKPT_BAD_HEADER = 2,
    MGV_CKPT_BAD_OFFSETS = 3,
    MGV_CKPT_IO = 4
} mgv_ckpt_error_kind; /* CheckpointError::Kind, same order */
const char* mgv_ckpt_last_error(void);
int mgv_ckpt_last_error_kind(void); /* -1 when the last error was not a CheckpointError */
mgv_status mgv_ckpt_load(const char* path, mgv_ckpt** out);
void mgv_ckpt_free(mgv_ckpt* ck);
int64_t mgv_ckpt_count(const mgv_ckpt* ck);
const char* mgv_ckpt_name(const mgv_ckpt* ck, int64_t i);
int mgv_ckpt_dtype(const mgv_ckpt* ck, int64_t i); /* mgv_ckpt_dtype_t */
int mgv_ckpt_rank(const mgv_ckpt* ck, int64_t i);
const int64_t* mgv_ckpt_shape(const mgv_ckpt* ck, int64_t i);
int64_t mgv_ckpt_numel(const mgv_ckpt* ck, int64_t i);
int64_t mgv_ckpt_find(const mgv_ckpt* ck, const char* name); /* -1 if absent */
/* widened to fp64 exactly as the reference loads it (f32 payloads -> double) */
mgv_status mgv_ckpt_read(const mgv_ckpt* ck, int64_t i, double* out);
int64_t mgv_ckpt_meta_count(const mgv_ckpt* ck);
const char* mgv_ckpt_meta_key(const mgv_ckpt* ck, int64_t i); /* sorted keys */
const char* mgv_ckpt_meta_value(const mgv_ckpt* ck, int64_t i);
/* save_checkpoint of n tensors (any order; dtypes NULL = all f64) plus string metadata.  MGV_ERR_INPUT for
 * the reserved name "__meta__" (params.cpp:93), duplicates or ill-formed UTF-8. */
mgv_status mgv_ckpt_save(const char* path, int64_t n, const char* const* names, const double* const* data,
                         const int* dtypes, const int* ranks, const int64_t* const* shapes, int64_t n_meta,
                         const char* const* meta_keys, const char* const* meta_values);
/* mgv_params_upload from a loaded checkpoint's dit.* entries: f32 payloads go to the device fp32 masters
 * bit-exactly, f64 payloads are rounded once (as mgv_params_upload does). */
mgv_status mgv_params_upload_ckpt(mgv_ctx* ctx, const mgv_dit_cfg* cfg, const mgv_ckpt* ck);
/* save_checkpoint of the context's dit.* parameters (e.g. after AdamW steps), dtype f32 (the fp32 masters,
 * bit-exact) or f64 (widened), with string metadata. */
mgv_status mgv_params_save(mgv_ctx* ctx, const char* path, int dtype, int64_t n_meta, const char* const* meta_keys,
                           const char* const* meta_values);

/* ---- Post-training on the same forward (proj/src/posttrain.cpp) ---- */
/* post::flow_error (posttrain.cpp:126-142) of n records, forward only: errs[k] = masked flow loss l_k. */
mgv_status mgv_flow_errors(mgv_ctx* ctx, int64_t n, const mgv_eval_sample* recs, double* errs);
/* One fwd+bwd over n records with Loss = sum_k weights[k] l_k: gradients sum_k w_k dl_k/dtheta, grad_norm
 * (flowtrain.cpp:284-289) and, when mgv_ctx_set_adamw is on, the AdamW update.  errs[k] = l_k, *loss = Loss. */
mgv_status mgv_flow_step_weighted(mgv_ctx* ctx, int64_t n, const mgv_eval_sample* recs, const double* weights,
                                  double* errs, double* loss, double* grad_norm, double* const* grads_out);

/* post::PostTrainConfig (posttrain.hpp:37-44); interleave = n_interleave tags, each "dpo" or "kto" */
typedef struct {
    double beta, alpha_sft, gamma_merge, w_d, w_u;
    int64_t n_interleave;
    const char* const* interleave;
} mgv_post_cfg;
/* post::SampleRecord (posttrain.hpp:15-21): latent rows on a grid, its ConditionMask, text and fps */
typedef struct {
    int64_t dims[3];
    const int32_t* coords;
    const double* rows;              /* N x 4c_z */
    const uint8_t* conditioned;      /* N flags or NULL */
    const double* condition_latents; /* N x 4c_z or NULL (= rows) */
    const double* text;              /* L x text_dim */
    int64_t L;
    double fps;
} mgv_sample_record;
typedef struct { mgv_sample_record winner, loser; } mgv_pref_pair;            /* posttrain.hpp:24-28 */
typedef struct { mgv_sample_record sample; int desirable; } mgv_labeled_sample; /* posttrain.hpp:30-33 */
typedef struct { double total, preference, sft, grad_norm; } mgv_post_metrics; /* posttrain.hpp:138-143 */
typedef struct mgv_post_state mgv_post_state;

/* post::validate(PostTrainConfig) (posttrain.cpp:37-49): MGV_ERR_CONFIG with the reference's message */
mgv_status mgv_post_validate(const mgv_post_cfg* cfg, char* err, int64_t err_cap);
/* PostTrainState(start, cfg, lr, seed) (posttrain.cpp:250-253): `policy` holds the trained weights (its AdamW is
 * set to AdamW(lr) defaults), `ref` the frozen reference copy (upload the same start weights to both). */
mgv_status mgv_post_state_create(mgv_ctx* policy, mgv_ctx* ref, double lr, uint64_t seed, mgv_post_state** out);
void mgv_post_state_destroy(mgv_post_state* st);
int64_t mgv_post_plan_pos(const mgv_post_state* st);
const char* mgv_post_last_error(const mgv_post_state* st);
/* post_train_step (posttrain.cpp:292-320): tag "dpo" consumes pairs, "kto" labels; the SFT batch is a
 * FlowBatch (flowtrain.hpp:111-123, shared text and fps).  Draws come from the state's Rng, as the
 * reference's make_pair_draws / make_label_draws.  MGV_ERR_SCHEDULING if tag != the plan's next tag. */
mgv_status mgv_post_train_step(mgv_post_state* st, const mgv_post_cfg* cfg, const char* tag, int64_t n_pairs,
                               const mgv_pref_pair* pairs, int64_t n_labels, const mgv_labeled_sample* labels,
                               int64_t n_sft, const mgv_flow_sample* sft, const double* sft_text, int64_t sft_L,
                               double sft_fps, mgv_post_metrics* out);
/* dpo_loss / kto_loss (posttrain.cpp:171-177, 224-233): the preference loss alone, forward only, with draws
 * from Rng(seed); kto uses cfg->beta, w_d, w_u. */
mgv_status mgv_post_pref_loss(mgv_ctx* policy, mgv_ctx* ref, const mgv_post_cfg* cfg, const char* tag,
                              int64_t n_pairs, const mgv_pref_pair* pairs, int64_t n_labels,
                              const mgv_labeled_sample* labels, uint64_t seed, double* loss);
/* post::rdpo_pairs (posttrain.cpp:235-254) on the device sampler: winners[k] / losers[k] (N_k x 4c_z) for record k:
 * winner = forward(reverse(rows)), loser = forward(fresh normals from Rng(seed), drawn record by record). */
mgv_status mgv_rdpo_pairs(mgv_ctx* ctx, int64_t n, const mgv_sample_record* recs, int64_t steps, uint64_t seed,
                          double* const* winners, double* const* losers);
/* post::merge_weights (k normalised weights gamma^(k-1-i)) and post::anneal_lr (cosine decay), posttrain.cpp:51-94 */
mgv_status mgv_merge_weights(int64_t k, double gamma, double* out);
mgv_status mgv_anneal_lr(int64_t step, double lr_start, double lr_end, int64_t steps, double* out);
/* scalar helpers: dpo_from_errors, kto_from_rewards (z0 NULL = batch mean) (posttrain.cpp:144-204) */
double mgv_dpo_from_errors(double e_th_w, double e_th_l, double e_ref_w, double e_ref_l, double beta);
mgv_status mgv_kto_from_rewards(int64_t n, const double* rewards, const uint8_t* desirable, double w_d, double w_u,
                                const double* z0_override, double* out);

#ifdef __cplusplus
}
#endif
#endif /* MUGV_B200_H */
