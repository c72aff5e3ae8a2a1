// extern "C" boundary (include/mugv_b200.h): C types only, no exceptions cross it.
#include <algorithm>
#include <cctype>
#include <cstring>
#include <exception>
#include <iterator>
#include <memory>
#include <string>

#include "ckpt.h"
#include "gemm.cuh"
#include "kernels.h"
#include "model.h"

#include "capi_internal.h"
#include "host_rng.h"

namespace {
// rmsnorm_rows (autodiff.cpp:686-701) of the looked-up text rows, one thread per row, the reference's
// sequential fp64 order without contraction: bit-identical to text_embed (dit.cpp:213-234)
__global__ void text_rms_kernel(const double* rows, int64_t L, int64_t D, double* out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= L) return;
    const double* r = rows + i * D;
    double ms = 0.0;
    for (int64_t j = 0; j < D; ++j) ms = __dadd_rn(ms, __dmul_rn(r[j], r[j]));
    ms = __ddiv_rn(ms, static_cast<double>(D));
    const double iv = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(ms, 1e-6)));  // kNormEps (dit.cpp:13)
    for (int64_t j = 0; j < D; ++j) out[i * D + j] = __dmul_rn(r[j], iv);
}

template <class F>
mgv_status guard(mgv_ctx* ctx, F&& f) {
    if (!ctx) return MGV_ERR_INPUT;
    return mgv::guard_into(ctx->err, std::forward<F>(f));
}
mgv::Cfg to_cfg(const mgv_dit_cfg* c) {
    mgv::Cfg g;
    g.depth = c->depth;
    g.hidden = c->hidden;
    g.heads = c->heads;
    g.text_dim = c->text_dim;
    g.c_z = c->c_z;
    for (int i = 0; i < 3; ++i) g.rope[i] = c->rope_split[i];
    return g;
}
}  // namespace

extern "C" {

mgv_status mgv_ctx_create(int device, int precision, mgv_ctx** out) {
    if (!out) return MGV_ERR_INPUT;
    *out = nullptr;
    auto* c = new mgv_ctx();
    mgv_status st = guard(c, [&] {
        if (precision != MGV_PREC_FP32 && precision != MGV_PREC_BF16) throw mgv::ConfigError("unknown precision");
        c->model = std::make_unique<mgv::Model>(device, precision == MGV_PREC_BF16);
    });
    if (st != MGV_OK) {
        delete c;
        return st;
    }
    *out = c;
    return MGV_OK;
}

void mgv_ctx_destroy(mgv_ctx* ctx) { delete ctx; }
const char* mgv_last_error(mgv_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

mgv_status mgv_ctx_set_stream(mgv_ctx* ctx, void* stream) {
    return guard(ctx, [&] { ctx->model->set_stream(static_cast<cudaStream_t>(stream)); });
}

mgv_status mgv_nccl_unique_id(uint8_t out[128]) {
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return MGV_ERR_NCCL;
    std::memcpy(out, &id, 128);
    return MGV_OK;
}

mgv_status mgv_ctx_set_dp(mgv_ctx* ctx, int rank, int world, const uint8_t nccl_id[128]) {
    return guard(ctx, [&] { ctx->model->set_dp(rank, world, nccl_id); });
}
mgv_status mgv_sample_rows(mgv_ctx* ctx, const double* x_start, int64_t N, const int32_t* coords,
                           const int64_t dims[3], const double* text, int64_t L, const uint8_t* conditioned,
                           const double* condition_latents, int64_t steps, int direction, double fps, double* out) {
    return guard(ctx, [&] {
        if (!x_start || !coords || !dims || !text || !out) throw mgv::InputError("null argument");
        if (direction != 1 && direction != -1) throw mgv::InputError("direction must be -1 (t 1->0) or +1 (t 0->1)");
        ctx->model->sample_rows(x_start, N, coords, dims, text, L, conditioned, condition_latents, steps, direction, fps,
                                out);
    });
}
mgv_status mgv_ctx_set_adamw(mgv_ctx* ctx, double lr, double beta1, double beta2, double eps, double weight_decay) {
    return guard(ctx, [&] { ctx->model->set_adamw(lr, beta1, beta2, eps, weight_decay); });
}
int64_t mgv_adamw_steps(mgv_ctx* ctx) { return ctx ? ctx->model->adamw_steps() : 0; }
mgv_status mgv_param_download(mgv_ctx* ctx, int64_t i, double* out) {
    return guard(ctx, [&] {
        if (!out) throw mgv::InputError("null output");
        ctx->model->download_param(i, out);
    });
}
mgv_status mgv_ctx_set_tp(mgv_ctx* ctx, int size, int rank, const uint8_t* nccl_id) {
    return guard(ctx, [&] { ctx->model->set_tp(size, rank, nccl_id); });
}

mgv_status mgv_params_upload(mgv_ctx* ctx, const mgv_dit_cfg* cfg, int64_t n, const char* const* names,
                             const double* const* data, const int64_t* numel) {
    return guard(ctx, [&] {
        if (!cfg) throw mgv::InputError("null config");
        ctx->model->upload(to_cfg(cfg), n, names, data, numel);
    });
}

// dit::init_dit_params (dit.cpp:143-183) drawn with mugv::Rng(seed) in the reference's order, then (gate_seed != 0)
// the gate-opening draws of the tests / SURVEY 8(d) from Rng(gate_seed): dit.mod.{w,b} and dit.final.w with std
// gate_std, dit.final.b with gate_b_std (test_dit.cpp:35-41).  Bit-identical weights to the reference's.
mgv_status mgv_params_init(mgv_ctx* ctx, const mgv_dit_cfg* cfg, uint64_t seed, uint64_t gate_seed, double gate_std,
                           double gate_b_std) {
    return guard(ctx, [&] {
        if (!cfg) throw mgv::InputError("null config");
        const mgv::Cfg c = to_cfg(cfg);
        mgv::validate_cfg(c);
        const int64_t H = c.hidden, D = c.D(), F = 32;  // kFreqDim (dit.cpp:15)
        std::vector<std::pair<std::string, std::vector<double>>> p;
        mgv::HostRng rng(seed);
        auto lin = [&](const std::string& n, int64_t out, int64_t in) {
            std::vector<double> w(static_cast<size_t>(out * in));
            rng.normal_fill(w.data(), out * in, 1.0 / std::sqrt(static_cast<double>(in)));
            p.emplace_back(n, std::move(w));
        };
        auto fill = [&](const std::string& n, int64_t k, double v) { p.emplace_back(n, std::vector<double>(k, v)); };
        lin("dit.patch.w", H, D);
        fill("dit.patch.b", H, 0.0);
        lin("dit.gmlp.in.w", H, F);
        fill("dit.gmlp.in.b", H, 0.0);
        lin("dit.gmlp.out.w", H, H);
        fill("dit.gmlp.out.b", H, 0.0);
        fill("dit.mod.w", 6 * H * H, 0.0);
        fill("dit.mod.b", 6 * H, 0.0);
        for (int64_t i = 0; i < c.depth; ++i) {
            const std::string b = "dit.blk." + std::to_string(i) + ".";
            fill(b + "gscale", H, 1.0);
            lin(b + "attn.qkv.w", 3 * H, H);
            fill(b + "attn.qkv.b", 3 * H, 0.0);
            fill(b + "attn.temp", c.heads, std::sqrt(static_cast<double>(c.hd())));
            lin(b + "attn.out.w", H, H);
            fill(b + "attn.out.b", H, 0.0);
            fill(b + "xattn.prenorm.g", H, 1.0);
            lin(b + "xattn.q.w", H, H);
            fill(b + "xattn.q.b", H, 0.0);
            lin(b + "xattn.kv.w", 2 * H, c.text_dim);
            fill(b + "xattn.kv.b", 2 * H, 0.0);
            lin(b + "xattn.out.w", H, H);
            fill(b + "xattn.out.b", H, 0.0);
            fill(b + "xattn.postnorm.g", H, 1.0);
            lin(b + "ffn.in.w", 4 * H, H);
            fill(b + "ffn.in.b", 4 * H, 0.0);
            lin(b + "ffn.out.w", H, 4 * H);
            fill(b + "ffn.out.b", H, 0.0);
        }
        fill("dit.final.g", H, 1.0);
        fill("dit.final.w", H * H, 0.0);
        fill("dit.final.b", H, 0.0);
        lin("dit.out.w", D, H);
        fill("dit.out.b", D, 0.0);
        if (gate_seed != 0) {  // open_gates: mod.w, mod.b, final.w, final.b in this order
            mgv::HostRng g(gate_seed);
            auto find = [&](const char* n) -> std::vector<double>& {
                for (auto& e : p)
                    if (e.first == n) return e.second;
                throw mgv::InputError(n);
            };
            const char* order[4] = {"dit.mod.w", "dit.mod.b", "dit.final.w", "dit.final.b"};
            for (int k = 0; k < 4; ++k) {
                std::vector<double>& v = find(order[k]);
                g.normal_fill(v.data(), static_cast<int64_t>(v.size()), k == 3 ? gate_b_std : gate_std);
            }
        }
        std::vector<const char*> names;
        std::vector<const double*> data;
        std::vector<int64_t> numel;
        for (auto& e : p) {
            names.push_back(e.first.c_str());
            data.push_back(e.second.data());
            numel.push_back(static_cast<int64_t>(e.second.size()));
        }
        ctx->model->upload(c, static_cast<int64_t>(names.size()), names.data(), data.data(), numel.data());
    });
}

// mugv::Rng(seed).uniform_tensor(n, lo, hi) (rng.hpp:60-64): the seeded synthetic latents of SURVEY 8(d)
mgv_status mgv_rng_uniform_fill(uint64_t seed, int64_t n, double lo, double hi, double* out) {
    if (!out || n < 0) return MGV_ERR_INPUT;
    mgv::HostRng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = lo + (hi - lo) * r.uniform();
    return MGV_OK;
}

// flow::make_batch (flowtrain.cpp:231-250) for one sample of N rows x D from Rng(seed): noise ~ N(0,1), t ~ U(0,1]
// (redrawn while <= 0), then the mask draw: *conditioned = uniform() < mask_prob (first_frame_mask)
mgv_status mgv_make_flow_sample(uint64_t seed, int64_t N, int64_t D, double mask_prob, double* noise, double* t,
                                int* conditioned) {
    if (!noise || !t || N < 0 || D < 1) return MGV_ERR_INPUT;
    mgv::HostRng r(seed);
    r.normal_fill(noise, N * D, 1.0);
    double u = r.uniform();
    while (u <= 0.0) u = r.uniform();
    *t = u;
    const bool c = r.uniform() < mask_prob;
    if (conditioned) *conditioned = c ? 1 : 0;
    return MGV_OK;
}

mgv_status mgv_ctx_set_varlen(mgv_ctx* ctx, int on) {
    return guard(ctx, [&] { ctx->model->set_varlen(on != 0); });
}

mgv_status mgv_ctx_set_recompute(mgv_ctx* ctx, int on) {
    return guard(ctx, [&] { ctx->model->set_recompute(on != 0); });
}

// per-rank memory of a training (or forward) step: {parameters, gradients, AdamW moments, workspace, exchange}
mgv_status mgv_plan_rank_bytes(const mgv_dit_cfg* cfg, int precision, int tp, int64_t N, int64_t L, int64_t n_u,
                               int train, int64_t out[5]) {
    std::string err;
    return mgv::guard_into(err, [&] {
        if (!cfg || !out || N < 1 || L < 1 || n_u < 1) throw mgv::InputError("bad argument");
        mgv::plan_rank_bytes(to_cfg(cfg), precision == MGV_PREC_BF16, tp, N, L, static_cast<int>(n_u),
                             train == 0 ? 0 : (train & 2) ? 3 : 1, out);
    });
}
mgv_status mgv_ctx_memory(mgv_ctx* ctx, int64_t out[5]) {
    return guard(ctx, [&] {
        if (!out) throw mgv::InputError("null argument");
        ctx->model->memory_bytes(out);
    });
}

mgv_status mgv_params_upload_ckpt(mgv_ctx* ctx, const mgv_dit_cfg* cfg, const mgv_ckpt* ck) {
    return guard(ctx, [&] {
        if (!cfg || !ck) throw mgv::InputError("null argument");
        // the payloads go to the device straight from the loaded file: little-endian f32 / f64 arrays that
        // cudaMemcpy reads at any alignment, so no host-side copy of the (possibly 10B-parameter) weights
        static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "MUGVCKPT payloads are little-endian");
        std::vector<const char*> names;
        std::vector<const void*> data;
        std::vector<uint8_t> is_f32;
        std::vector<int64_t> numel;
        for (const mgv::CkptEntry& e : ck->ck.entries) {
            if (e.name.rfind("dit.", 0) != 0) continue;  // register_params(..., "dit.") (flowtrain.cpp:260)
            names.push_back(e.name.c_str());
            numel.push_back(e.numel);
            is_f32.push_back(e.dtype == mgv::kF32);
            data.push_back(ck->ck.payload(e));
        }
        ctx->model->upload(to_cfg(cfg), static_cast<int64_t>(names.size()), names.data(), data.data(), is_f32.data(),
                           numel.data());
    });
}

mgv_status mgv_params_save(mgv_ctx* ctx, const char* path, int dtype, int64_t n_meta, const char* const* meta_keys,
                           const char* const* meta_values) {
    return guard(ctx, [&] {
        if (!path || (n_meta > 0 && (!meta_keys || !meta_values))) throw mgv::InputError("null argument");
        if (dtype != MGV_CKPT_F32 && dtype != MGV_CKPT_F64) throw mgv::InputError("unknown dtype");
        const auto& ps = ctx->model->sorted_params();
        if (ps.empty()) throw mgv::InputError("no parameters uploaded");
        std::vector<std::vector<double>> host(ps.size());
        std::vector<mgv::CkptTensorIn> ts(ps.size());
        for (size_t k = 0; k < ps.size(); ++k) {
            host[k].resize(static_cast<size_t>(ps[k]->numel_full));
            ctx->model->download_param(static_cast<int64_t>(k), host[k].data());  // fp32 master, widened exactly
            ts[k].name = ps[k]->name;
            ts[k].dtype = dtype == MGV_CKPT_F32 ? mgv::kF32 : mgv::kF64;
            ts[k].shape = ps[k]->shape;
            ts[k].f64 = host[k].data();
        }
        std::map<std::string, std::string> meta;
        for (int64_t k = 0; k < n_meta; ++k) {
            if (!meta_keys[k] || !meta_values[k]) throw mgv::InputError("null metadata argument");
            meta[meta_keys[k]] = meta_values[k];
        }
        mgv::save_checkpoint(std::move(ts), meta, path);
    });
}

int64_t mgv_param_count(mgv_ctx* ctx) { return ctx ? static_cast<int64_t>(ctx->model->sorted_params().size()) : 0; }
const char* mgv_param_name(mgv_ctx* ctx, int64_t i) { return ctx->model->sorted_params()[i]->name.c_str(); }
int64_t mgv_param_numel(mgv_ctx* ctx, int64_t i) { return ctx->model->sorted_params()[i]->numel_full; }

mgv_status mgv_predict_velocity(mgv_ctx* ctx, const double* rows, int64_t N, const int32_t* coords,
                                const int64_t dims[3], const double* text, int64_t L, const double* timesteps,
                                double fps, double* out) {
    return guard(ctx, [&] { ctx->model->predict_velocity(rows, N, coords, dims, text, L, timesteps, fps, out); });
}

mgv_status mgv_velocity_graph(mgv_ctx* ctx, const double* rows, int64_t N, const int32_t* coords,
                              const int64_t dims[3], const double* text, int64_t L, const double* timesteps,
                              double fps, double* velocity, double* const* taps, const double* dV,
                              double* const* grads_out) {
    return guard(ctx, [&] {
        ctx->model->velocity_graph(rows, N, coords, dims, text, L, timesteps, fps, velocity, taps, dV, grads_out);
    });
}

mgv_status mgv_dit_forward(mgv_ctx* ctx, const double* tokens, int64_t N, const int32_t* coords,
                           const int64_t dims[3], const double* text, int64_t L, const double* timesteps, double fps,
                           double* out) {
    return guard(ctx, [&] { ctx->model->dit_forward(tokens, N, coords, dims, text, L, timesteps, fps, out); });
}

int64_t mgv_tokenize(const char* prompt, int64_t vocab, int64_t* ids, int64_t cap) {
    // dit::tokenize (dit.cpp:193-211): whitespace-split words, FNV-1a 64 of each, modulo the vocabulary
    if (!prompt || vocab < 1) return -1;
    int64_t n = 0;
    size_t i = 0;
    const std::string s(prompt);
    while (i < s.size()) {
        while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
        size_t j = i;
        while (j < s.size() && !std::isspace(static_cast<unsigned char>(s[j]))) ++j;
        if (j > i) {
            uint64_t h = 1469598103934665603ull;
            for (size_t k = i; k < j; ++k) {
                h ^= static_cast<unsigned char>(s[k]);
                h *= 1099511628211ull;
            }
            if (ids && n < cap) ids[n] = static_cast<int64_t>(h % static_cast<uint64_t>(vocab));
            ++n;
        }
        i = j;
    }
    return n;
}

mgv_status mgv_text_embed(mgv_ctx* ctx, const int64_t* ids, int64_t n, const double* embed_table, int64_t vocab,
                          const double* null_row, int64_t text_dim, int64_t max_len, double* out, int* truncated) {
    return guard(ctx, [&] {
        if (n < 0 || (n > 0 && !ids) || !embed_table || !null_row || !out || text_dim < 1 || max_len < 1)
            throw mgv::InputError("bad text_embed arguments");
        const int64_t use = std::min(n, max_len);  // truncate first (dit.cpp:225-229)
        if (truncated) *truncated = n > max_len ? 1 : 0;
        for (int64_t k = 0; k < use; ++k)
            if (ids[k] < 0 || ids[k] >= vocab)
                throw mgv::InputError("text id " + std::to_string(ids[k]) + " outside the vocabulary");  // :214-216
        const int64_t L = use > 0 ? use : 1;  // empty -> the learned null row
        std::vector<double> rows(static_cast<size_t>(L * text_dim));
        for (int64_t k = 0; k < L; ++k)
            std::memcpy(rows.data() + k * text_dim, use > 0 ? embed_table + ids[k] * text_dim : null_row,
                        sizeof(double) * text_dim);
        cudaStream_t s = ctx->model->stream();
        double *dr = nullptr, *dout = nullptr;
        MGV_CUDA(cudaMallocAsync(&dr, sizeof(double) * L * text_dim, s));
        MGV_CUDA(cudaMallocAsync(&dout, sizeof(double) * L * text_dim, s));
        MGV_CUDA(cudaMemcpyAsync(dr, rows.data(), sizeof(double) * L * text_dim, cudaMemcpyHostToDevice, s));
        text_rms_kernel<<<static_cast<unsigned>((L + 63) / 64), 64, 0, s>>>(dr, L, text_dim, dout);
        mgv::note_launch();
        MGV_CUDA(cudaGetLastError());
        MGV_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * L * text_dim, cudaMemcpyDeviceToHost, s));
        MGV_CUDA(cudaFreeAsync(dr, s));
        MGV_CUDA(cudaFreeAsync(dout, s));
        MGV_CUDA(cudaStreamSynchronize(s));
    });
}

mgv_status mgv_patchify(mgv_ctx* ctx, const double* grid, int64_t U, int64_t h, int64_t w, int64_t C, double* tokens,
                        int32_t* coords) {
    return guard(ctx, [&] { ctx->model->patchify(grid, U, h, w, C, tokens, coords); });
}
mgv_status mgv_unpatchify(mgv_ctx* ctx, const double* tokens, int64_t N, const int32_t* coords, const int64_t dims[3],
                          double* grid) {
    return guard(ctx, [&] { ctx->model->unpatchify(tokens, N, coords, dims, grid); });
}
mgv_status mgv_global_embed(mgv_ctx* ctx, const double* timesteps, int64_t N, double fps, double* g,
                            double* block_scales) {
    return guard(ctx, [&] { ctx->model->global_embed_host(timesteps, N, fps, g, block_scales); });
}

mgv_status mgv_fused_modulate(mgv_ctx* ctx, const double* x, const double* bias, int64_t bias_n, const double* scale,
                              int64_t scale_n, const double* shift, int64_t shift_n, const double* residual,
                              int64_t rows, int64_t cols, double* out) {
    return guard(ctx, [&] {
        mgv::fused_modulate_host(x, bias, bias_n, scale, scale_n, shift, shift_n, residual, rows, cols, out,
                                 ctx->model->stream());
    });
}
mgv_status mgv_dev_fused_modulate_f32(mgv_ctx* ctx, const float* x, const float* bias, const float* scale,
                                      const float* shift, const float* residual, int64_t rows, int64_t cols,
                                      float* out) {
    return guard(ctx, [&] {
        mgv::fused_modulate_dev_f32(x, bias, scale, shift, residual, rows, cols, out, ctx->model->stream());
    });
}
mgv_status mgv_apply_rope3d(mgv_ctx* ctx, const double* x, int64_t N, int64_t heads, const int64_t split[3],
                            const int32_t* coords, double base, int inverse, double* out) {
    return guard(ctx, [&] {
        mgv::apply_rope3d_host(x, N, heads, split, coords, base, inverse, out, ctx->model->stream());
    });
}

mgv_status mgv_flow_step(mgv_ctx* ctx, int64_t n, const mgv_flow_sample* samples, const double* text, int64_t L,
                         double fps, double* loss, double* grad_norm, double* const* grads_out,
                         double* const* velocity_out) {
    return guard(ctx, [&] {
        ctx->model->flow_step(n, samples, text, L, fps, loss, grad_norm, grads_out, velocity_out);
    });
}

// Device-resident variant for the benchmark's `value` figure (pointers in `samples` are device pointers).
mgv_status mgv_flow_step_device(mgv_ctx* ctx, int64_t n, const mgv_flow_sample* samples, const double* text_dev,
                                int64_t L, double fps, double* loss, double* grad_norm) {
    return guard(ctx, [&] {
        std::vector<mgv::DevSample> ds(static_cast<size_t>(n));
        for (int64_t k = 0; k < n; ++k) {
            const mgv_flow_sample& s = samples[k];
            mgv::DevSample& d = ds[static_cast<size_t>(k)];
            d.N = s.dims[0] * s.dims[1] * s.dims[2];
            std::memcpy(d.dims, s.dims, sizeof(d.dims));
            d.coords = s.coords;
            d.clean = s.clean_rows;
            d.noise = s.noise;
            d.t = s.t;
            d.cond = s.conditioned;  // device flags (caller-validated, unit-aligned) or null
            d.cond_lat = s.condition_latents;
        }
        ctx->model->flow_step_dev(n, ds.data(), text_dev, L, fps, loss, grad_norm);
    });
}

mgv_status mgv_flow_loss(mgv_ctx* ctx, const double* pred, const double* target, const uint8_t* mask, int64_t N,
                         int64_t D, double* loss) {
    // flowtrain.cpp:22-38: tiny host-side reduction API kept for drop-in completeness
    return guard(ctx, [&] {
        if (!pred || !target || !mask || N < 0 || D < 1) throw mgv::DimensionError("flow_loss needs (N, D) rows");
        double sum = 0.0;
        int64_t count = 0;
        for (int64_t i = 0; i < N; ++i) {
            if (!mask[i]) continue;
            for (int64_t j = 0; j < D; ++j) {
                const double d = pred[i * D + j] - target[i * D + j];
                sum += d * d;
            }
            count += D;
        }
        *loss = count > 0 ? sum / static_cast<double>(count) : 0.0;
    });
}

mgv_status mgv_latent_rows(mgv_ctx* ctx, const double* grid, int64_t U, int64_t h, int64_t w, int64_t C,
                           double* rows, int32_t* coords) {
    return guard(ctx, [&] {
        if (U < 1 || h < 1 || w < 1 || C < 1) throw mgv::DimensionError("latent grid must be (U, h, w, C)");
        if (h % 2 != 0 || w % 2 != 0) throw mgv::DimensionError("patchify needs even spatial dims");  // dit.cpp:95
        cudaStream_t s = ctx->model->stream();
        const int64_t n_in = U * h * w * C, N = U * (h / 2) * (w / 2);
        double *dg = nullptr, *dr = nullptr;
        int32_t* dc = nullptr;
        MGV_CUDA(cudaMallocAsync(&dg, sizeof(double) * n_in, s));
        MGV_CUDA(cudaMallocAsync(&dr, sizeof(double) * n_in, s));
        MGV_CUDA(cudaMallocAsync(&dc, sizeof(int32_t) * 3 * N, s));
        MGV_CUDA(cudaMemcpyAsync(dg, grid, sizeof(double) * n_in, cudaMemcpyHostToDevice, s));
        mgv::latent_rows_gather(dg, int(U), int(h), int(w), int(C), dr, dc, s);
        MGV_CUDA(cudaMemcpyAsync(rows, dr, sizeof(double) * n_in, cudaMemcpyDeviceToHost, s));
        MGV_CUDA(cudaMemcpyAsync(coords, dc, sizeof(int32_t) * 3 * N, cudaMemcpyDeviceToHost, s));
        MGV_CUDA(cudaFreeAsync(dg, s));
        MGV_CUDA(cudaFreeAsync(dr, s));
        MGV_CUDA(cudaFreeAsync(dc, s));
        MGV_CUDA(cudaStreamSynchronize(s));
    });
}

mgv_status mgv_rows_to_grid(mgv_ctx* ctx, const double* rows, const int32_t* coords, int64_t N, const int64_t dims[3],
                            int64_t C, double* grid) {
    return guard(ctx, [&] {
        if (N != dims[0] * dims[1] * dims[2]) throw mgv::DimensionError("token coords do not match the grid dims");
        cudaStream_t s = ctx->model->stream();
        const int64_t n = N * 4 * C;
        double *dr = nullptr, *dg = nullptr;
        int32_t *dc = nullptr, *seen = nullptr, *st = nullptr;
        MGV_CUDA(cudaMallocAsync(&dr, sizeof(double) * n, s));
        MGV_CUDA(cudaMallocAsync(&dg, sizeof(double) * n, s));
        MGV_CUDA(cudaMallocAsync(&dc, sizeof(int32_t) * 3 * N, s));
        MGV_CUDA(cudaMallocAsync(&seen, sizeof(int32_t) * N, s));
        MGV_CUDA(cudaMallocAsync(&st, sizeof(int32_t), s));
        MGV_CUDA(cudaMemcpyAsync(dr, rows, sizeof(double) * n, cudaMemcpyHostToDevice, s));
        MGV_CUDA(cudaMemcpyAsync(dc, coords, sizeof(int32_t) * 3 * N, cudaMemcpyHostToDevice, s));
        MGV_CUDA(cudaMemsetAsync(dg, 0, sizeof(double) * n, s));
        mgv::rows_to_grid_scatter(dr, dc, int(N), int(dims[0]), int(dims[1]), int(dims[2]), int(C), dg, seen, st, s);
        int32_t status = 0;
        MGV_CUDA(cudaMemcpyAsync(&status, st, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        MGV_CUDA(cudaMemcpyAsync(grid, dg, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
        MGV_CUDA(cudaFreeAsync(dr, s));
        MGV_CUDA(cudaFreeAsync(dg, s));
        MGV_CUDA(cudaFreeAsync(dc, s));
        MGV_CUDA(cudaFreeAsync(seen, s));
        MGV_CUDA(cudaFreeAsync(st, s));
        MGV_CUDA(cudaStreamSynchronize(s));
        if (status == 1) throw mgv::DimensionError("token coord outside the grid");  // dit.cpp:129-130
        if (status == 2) throw mgv::DimensionError("duplicate token coord");         // dit.cpp:132
    });
}

double mgv_last_step_ms(mgv_ctx* ctx) { return ctx ? ctx->model->last_step_ms() : 0.0; }
int64_t mgv_last_step_launches(mgv_ctx* ctx) { return ctx ? ctx->model->last_step_launches() : 0; }

// Per-phase device timing for the benchmark (CUDA events on the context stream).
mgv_status mgv_prof_enable(mgv_ctx* ctx, int on) {
    return guard(ctx, [&] {
        ctx->model->prof().on = on != 0;
        ctx->model->prof().stats.clear();
    });
}
int64_t mgv_prof_count(mgv_ctx* ctx) { return ctx ? static_cast<int64_t>(ctx->model->prof().stats.size()) : 0; }
const char* mgv_prof_entry(mgv_ctx* ctx, int64_t i, double* ms, int64_t* n) {
    auto it = ctx->model->prof().stats.begin();
    std::advance(it, i);
    *ms = it->second.ms;
    *n = it->second.n;
    return it->first.c_str();
}
double mgv_prof_entry_work(mgv_ctx* ctx, int64_t i) {
    auto it = ctx->model->prof().stats.begin();
    std::advance(it, i);
    return it->second.work;
}

}  // extern "C"
