// ORACLE — TEST INFRASTRUCTURE ONLY (checker / CPU baseline, never the product).
//
// A thin extern "C" veneer over the UNMODIFIED reference library, compiled from
// the reference sources where they lie (/root/reference/proj/src, see
// oracle/Makefile) into oracle/_ref/libmugv_ref.so.  Python tests and bench.py's
// reference arm drive it through ctypes.  Every entry point calls the
// reference's own public API:
//   - dit::init_dit_params                       proj/src/dit.cpp:143-183
//   - open_gates-style gate randomisation        proj/tests/test_dit.cpp:35-41
//   - flow::interpolate / apply_condition_mask   proj/src/flowtrain.cpp:9-20,83-100
//   - dit::velocity_rows_graph (+taps)           proj/src/dit.cpp:320-334
//   - flow::flow_loss_graph, Tape::backward      proj/src/flowtrain.cpp:40-42, autodiff.cpp:82-92
//   - the per-sample loop of FlowTrainer::step   proj/src/flowtrain.cpp:257-279 (minus AdamW)
//   - dit::predict_velocity / dit::dit_forward   proj/src/dit.cpp:361-396
//   - flow::make_batch                           proj/src/flowtrain.cpp:231-250
//   - save_checkpoint / load_checkpoint          proj/src/params.cpp:92-225
//   - post::post_loss_graph (+ backward), make_pair_draws / make_label_draws, dpo_loss / kto_loss
//                                                proj/src/posttrain.cpp:106-290
#include <array>
#include <cmath>
#include <cstring>
#include <iterator>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "mugv/autodiff.hpp"
#include "mugv/optim.hpp"
#include "mugv/dit.hpp"
#include "mugv/flowtrain.hpp"
#include "mugv/params.hpp"
#include "mugv/posttrain.hpp"

using namespace mugv;

namespace {

thread_local std::string g_err;
thread_local int g_ckpt_kind = -1;

struct RefCfg {
    int64_t depth, hidden, heads, text_dim, c_z;
    int32_t rope[3];
};

dit::DitConfig to_cfg(const RefCfg* c) {
    dit::DitConfig cfg;
    cfg.depth = c->depth;
    cfg.hidden = c->hidden;
    cfg.heads = c->heads;
    cfg.text_dim = c->text_dim;
    cfg.c_z = c->c_z;
    cfg.rope_split = {c->rope[0], c->rope[1], c->rope[2]};
    return cfg;
}

struct Handle {
    ParameterSet p;
    std::vector<std::string> names;
    void refresh() { names = p.names(); }
};

dit::TokenGrid geom_of(const int64_t* d, int64_t c_z) {
    // grid_geom from proj/tests/test_flow.cpp:35-37: coords/dims only
    return dit::latent_rows(Tensor::zeros({d[0], 2 * d[1], 2 * d[2], c_z}));
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const DimensionError& e) {
        g_err = e.what();
        return 1;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const InputError& e) {
        g_err = e.what();
        return 3;
    } catch (const NumericError& e) {
        g_err = e.what();
        return 4;
    } catch (const CheckpointError& e) {
        g_err = e.what();
        g_ckpt_kind = static_cast<int>(e.kind);
        return 8;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_last_ckpt_kind() { return g_ckpt_kind; }

// ---- checkpoint container (params.cpp:92-225) ----
// dtypes: 0 = f32, 1 = f64 (Dtype order of params.hpp:14)
int ref_ckpt_save(const char* path, int64_t n, const char* const* names, const double* const* data, const int* dtypes,
                  const int* ranks, const int64_t* const* shapes, int64_t n_meta, const char* const* keys,
                  const char* const* values) {
    g_ckpt_kind = -1;
    return guard([&] {
        ParameterSet ps;
        for (int64_t k = 0; k < n; ++k) {
            std::vector<int64_t> shape(shapes[k], shapes[k] + ranks[k]);
            Tensor t(shape);
            std::memcpy(t.data(), data[k], sizeof(double) * static_cast<size_t>(t.numel()));
            ps.set(names[k], std::move(t), dtypes[k] == 0 ? Dtype::f32 : Dtype::f64);
        }
        for (int64_t k = 0; k < n_meta; ++k) ps.metadata[keys[k]] = values[k];
        save_checkpoint(ps, path);
    });
}
void* ref_ckpt_load(const char* path) {
    g_ckpt_kind = -1;
    Handle* h = nullptr;
    guard([&] {
        auto hh = std::make_unique<Handle>();
        hh->p = load_checkpoint(path);
        hh->refresh();
        h = hh.release();
    });
    return h;
}
int ref_params_dtype(void* h, int64_t i) {
    auto* hh = static_cast<Handle*>(h);
    return hh->p.entry(hh->names[static_cast<size_t>(i)]).dtype == Dtype::f32 ? 0 : 1;
}
int ref_params_rank(void* h, int64_t i) {
    auto* hh = static_cast<Handle*>(h);
    return static_cast<int>(hh->p.at(hh->names[static_cast<size_t>(i)]).shape().size());
}
const int64_t* ref_params_shape(void* h, int64_t i) {
    auto* hh = static_cast<Handle*>(h);
    return hh->p.at(hh->names[static_cast<size_t>(i)]).shape().data();
}
int64_t ref_params_meta_count(void* h) { return static_cast<int64_t>(static_cast<Handle*>(h)->p.metadata.size()); }
const char* ref_params_meta(void* h, int64_t i, int value) {
    auto it = static_cast<Handle*>(h)->p.metadata.begin();
    std::advance(it, i);
    return value ? it->second.c_str() : it->first.c_str();
}

// ---- Rng pins ----
void ref_rng_normal_fill(uint64_t seed, int64_t skip_uniform, int64_t n, double stddev, double* out) {
    Rng r(seed);
    for (int64_t i = 0; i < skip_uniform; ++i) r.uniform();
    Tensor t = r.normal_tensor({n}, stddev);
    std::memcpy(out, t.data(), sizeof(double) * static_cast<size_t>(n));
}

void ref_rng_uniform_fill(uint64_t seed, int64_t n, double lo, double hi, double* out) {
    Rng r(seed);
    Tensor t = r.uniform_tensor({n}, lo, hi);
    std::memcpy(out, t.data(), sizeof(double) * static_cast<size_t>(n));
}

// ---- parameters ----
void* ref_params_create(const RefCfg* c, uint64_t seed, int open_gates, uint64_t gate_seed, double gate_std,
                        double gate_b_std) {
    Handle* h = nullptr;
    int rc = guard([&] {
        auto cfg = to_cfg(c);
        Rng r(seed);
        auto hh = std::make_unique<Handle>();
        hh->p = dit::init_dit_params(cfg, r);
        if (open_gates) {
            Rng g(gate_seed);
            hh->p.at("dit.mod.w") = g.normal_tensor(hh->p.at("dit.mod.w").shape(), gate_std);
            hh->p.at("dit.mod.b") = g.normal_tensor(hh->p.at("dit.mod.b").shape(), gate_std);
            hh->p.at("dit.final.w") = g.normal_tensor(hh->p.at("dit.final.w").shape(), gate_std);
            hh->p.at("dit.final.b") = g.normal_tensor(hh->p.at("dit.final.b").shape(), gate_b_std);
        }
        hh->refresh();
        h = hh.release();
    });
    return rc == 0 ? h : nullptr;
}

void ref_params_destroy(void* h) { delete static_cast<Handle*>(h); }
int64_t ref_params_count(void* h) { return static_cast<int64_t>(static_cast<Handle*>(h)->names.size()); }
const char* ref_params_name(void* h, int64_t i) { return static_cast<Handle*>(h)->names[static_cast<size_t>(i)].c_str(); }
int64_t ref_params_numel(void* h, int64_t i) {
    auto* hh = static_cast<Handle*>(h);
    return hh->p.at(hh->names[static_cast<size_t>(i)]).numel();
}
double* ref_params_data(void* h, int64_t i) {
    auto* hh = static_cast<Handle*>(h);
    return hh->p.at(hh->names[static_cast<size_t>(i)]).data();
}

// ---- make_batch pin (flowtrain.cpp:231-250) ----
// grids: n pointers to (U,h,w,c_z) tensors with dims[3*i..]; outputs noise rows (N,4c_z), t, masked flag.
int ref_make_batch(int64_t n, const int64_t* dims, int64_t c_z, const double* const* grids, double fps,
                   double mask_prob, uint64_t seed, double* const* noise_out, double* t_out, int32_t* masked_out) {
    return guard([&] {
        std::vector<Tensor> gs;
        for (int64_t i = 0; i < n; ++i) {
            const int64_t* d = dims + 3 * i;
            Tensor g({d[0], d[1], d[2], c_z});
            std::memcpy(g.data(), grids[i], sizeof(double) * static_cast<size_t>(g.numel()));
            gs.push_back(std::move(g));
        }
        Rng r(seed);
        flow::FlowBatch b = flow::make_batch(gs, Tensor::zeros({1, 1}), fps, mask_prob, r);
        for (int64_t i = 0; i < n; ++i) {
            const auto& s = b.samples[static_cast<size_t>(i)];
            std::memcpy(noise_out[i], s.noise.data(), sizeof(double) * static_cast<size_t>(s.noise.numel()));
            t_out[i] = s.t;
            masked_out[i] = s.mask.any() ? 1 : 0;
        }
    });
}

// ---- the hot path: FlowTrainer::step forward + backward (no AdamW) ----
// dims: n x (U, Hp, Wp); clean/noise: (N_i, 4c_z) rows; cond: n x {0,1} first-frame flag.
// V_out[i] (N_i, 4c_z) and taps_out[i] ((depth+3) tensors concatenated: patch emb (N,H),
// block outputs (N,H) x depth, final proj (N,H), velocity (N,4c_z)) may be null.
// grads_out: one pointer per parameter in sorted-name order, or null.
// masks / cond_lat (both may be null): per-sample general ConditionMask flags (N_i bytes) and condition latents
// (N_i x 4c_z); a null masks[i] falls back to cond[i] (first_frame_mask).
int ref_flow_fwdbwd_masked(void* h, const RefCfg* c, int64_t n, const int64_t* dims, const double* const* clean,
                           const double* const* noise, const double* t, const int32_t* cond,
                           const uint8_t* const* masks, const double* const* cond_lat, const double* text, int64_t L,
                           double fps, double* loss_out, double* const* V_out, double* const* taps_out,
                           double* const* grads_out) {
    return guard([&] {
        auto* hh = static_cast<Handle*>(h);
        auto cfg = to_cfg(c);
        dit::validate(cfg);
        Tensor text_t({L, cfg.text_dim});
        std::memcpy(text_t.data(), text, sizeof(double) * static_cast<size_t>(text_t.numel()));
        Tape tp;
        ParamVars pv = register_params(tp, hh->p, grads_out != nullptr, "dit.");
        Var tx = tp.constant(text_t);
        Var total;
        std::vector<std::vector<Var>> all_taps(static_cast<size_t>(n));
        std::vector<Var> vs;
        for (int64_t i = 0; i < n; ++i) {
            dit::TokenGrid geom = geom_of(dims + 3 * i, cfg.c_z);
            int64_t N = geom.n(), D = cfg.patch_dim();
            Tensor cr({N, D}), nz({N, D});
            std::memcpy(cr.data(), clean[i], sizeof(double) * static_cast<size_t>(N * D));
            std::memcpy(nz.data(), noise[i], sizeof(double) * static_cast<size_t>(N * D));
            flow::ConditionMask mask = cond[i] ? flow::first_frame_mask(geom, cr) : flow::no_condition(N);
            if (masks && masks[i]) {
                mask.conditioned.assign(masks[i], masks[i] + N);
                mask.condition_latents = Tensor({N, D});
                std::memcpy(mask.condition_latents.data(), cond_lat && cond_lat[i] ? cond_lat[i] : clean[i],
                            sizeof(double) * static_cast<size_t>(N * D));
            }
            flow::Interpolated ip = flow::interpolate(cr, nz, t[i]);
            Tensor ts = Tensor::full({N}, t[i]);
            flow::MaskedInput mi = flow::apply_condition_mask(ip.x_t, ts, mask, geom);
            Var v = dit::velocity_rows_graph(tp, tp.constant(mi.rows), geom, tx, mi.timesteps, fps, pv, cfg,
                                             taps_out ? &all_taps[static_cast<size_t>(i)] : nullptr);
            vs.push_back(v);
            Var l = flow::flow_loss_graph(tp, v, ip.v_target, mi.loss_mask);
            total = (i == 0) ? l : tp.add(total, l);
        }
        total = tp.scale(total, 1.0 / static_cast<real>(n));
        *loss_out = tp.val(total)[0];
        for (int64_t i = 0; i < n; ++i) {
            if (V_out && V_out[i]) {
                const Tensor& V = tp.val(vs[static_cast<size_t>(i)]);
                std::memcpy(V_out[i], V.data(), sizeof(double) * static_cast<size_t>(V.numel()));
            }
            if (taps_out && taps_out[i]) {
                double* dst = taps_out[i];
                for (Var tv : all_taps[static_cast<size_t>(i)]) {
                    const Tensor& T = tp.val(tv);
                    std::memcpy(dst, T.data(), sizeof(double) * static_cast<size_t>(T.numel()));
                    dst += T.numel();
                }
            }
        }
        if (grads_out) {
            if (!std::isfinite(*loss_out)) throw NumericError("flow loss is not finite");
            tp.backward(total);
            auto grads = collect_grads(tp, pv);
            size_t k = 0;
            for (const auto& nm : hh->names) {
                if (grads_out[k]) {
                    const Tensor& g = grads.at(nm);
                    std::memcpy(grads_out[k], g.data(), sizeof(double) * static_cast<size_t>(g.numel()));
                }
                ++k;
            }
        }
    });
}

int ref_flow_fwdbwd(void* h, const RefCfg* c, int64_t n, const int64_t* dims, const double* const* clean,
                    const double* const* noise, const double* t, const int32_t* cond, const double* text, int64_t L,
                    double fps, double* loss_out, double* const* V_out, double* const* taps_out,
                    double* const* grads_out) {
    return ref_flow_fwdbwd_masked(h, c, n, dims, clean, noise, t, cond, nullptr, nullptr, text, L, fps, loss_out, V_out,
                                  taps_out, grads_out);
}

// predict_velocity (dit.cpp:388-396) on a row-major grid of dims (U,Hp,Wp).
int ref_predict_velocity(void* h, const RefCfg* c, const int64_t* dims, const double* rows, const double* tau,
                         const double* text, int64_t L, double fps, double* out) {
    return guard([&] {
        auto* hh = static_cast<Handle*>(h);
        auto cfg = to_cfg(c);
        dit::TokenGrid geom = geom_of(dims, cfg.c_z);
        int64_t N = geom.n();
        Tensor r({N, cfg.patch_dim()}), ts({N}), tx({L, cfg.text_dim});
        std::memcpy(r.data(), rows, sizeof(double) * static_cast<size_t>(r.numel()));
        std::memcpy(ts.data(), tau, sizeof(double) * static_cast<size_t>(N));
        std::memcpy(tx.data(), text, sizeof(double) * static_cast<size_t>(tx.numel()));
        Tensor v = dit::predict_velocity(r, geom, tx, ts, fps, hh->p, cfg);
        std::memcpy(out, v.data(), sizeof(double) * static_cast<size_t>(v.numel()));
    });
}

// dit_forward (dit.cpp:361-375): tokens (N, hidden) in, (N, hidden) out.
int ref_dit_forward(void* h, const RefCfg* c, const int64_t* dims, const double* tokens, const double* tau,
                    const double* text, int64_t L, double fps, double* out) {
    return guard([&] {
        auto* hh = static_cast<Handle*>(h);
        auto cfg = to_cfg(c);
        dit::TokenGrid geom = geom_of(dims, cfg.c_z);
        int64_t N = geom.n();
        geom.tokens = Tensor({N, cfg.hidden});
        std::memcpy(geom.tokens.data(), tokens, sizeof(double) * static_cast<size_t>(N * cfg.hidden));
        Tensor ts({N}), tx({L, cfg.text_dim});
        std::memcpy(ts.data(), tau, sizeof(double) * static_cast<size_t>(N));
        std::memcpy(tx.data(), text, sizeof(double) * static_cast<size_t>(tx.numel()));
        dit::TokenGrid o = dit::dit_forward(geom, tx, dit::GlobalSignals{ts, fps}, hh->p, cfg);
        std::memcpy(out, o.tokens.data(), sizeof(double) * static_cast<size_t>(o.tokens.numel()));
    });
}

// ---- sampler: forward_sample_rows (direction -1) / reverse_sample_rows (+1), flowtrain.cpp:135-172, with
// model_velocity (:102-107) on the handle's parameters; cond may be null (no_condition)
int ref_sample_rows(void* h, const RefCfg* c, const int64_t* dims, const double* x_start, const double* text,
                    int64_t L, const uint8_t* cond, const double* cond_latents, int64_t steps, int direction,
                    double fps, double* out) {
    return guard([&] {
        auto* hh = static_cast<Handle*>(h);
        auto cfg = to_cfg(c);
        dit::TokenGrid geom = geom_of(dims, cfg.c_z);
        const int64_t N = geom.n(), D = cfg.patch_dim();
        Tensor x({N, D}), tx({L, cfg.text_dim});
        std::memcpy(x.data(), x_start, sizeof(double) * static_cast<size_t>(x.numel()));
        std::memcpy(tx.data(), text, sizeof(double) * static_cast<size_t>(tx.numel()));
        flow::ConditionMask mask = flow::no_condition(N);
        if (cond) {
            mask.conditioned.assign(cond, cond + N);
            mask.condition_latents = Tensor({N, D});
            std::memcpy(mask.condition_latents.data(), cond_latents, sizeof(double) * static_cast<size_t>(N * D));
        }
        auto vel = flow::model_velocity(hh->p, cfg, geom, tx, fps);
        Tensor y = direction < 0 ? flow::forward_sample_rows(vel, geom, x, mask, steps)
                                 : flow::reverse_sample_rows(vel, geom, x, mask, steps);
        std::memcpy(out, y.data(), sizeof(double) * static_cast<size_t>(y.numel()));
    });
}

// ---- AdamW::update (optim.cpp:7-24) on caller-owned tensors ----
void* ref_adamw_create(double lr, double beta1, double beta2, double eps, double weight_decay) {
    auto* o = new AdamW(lr);
    o->beta1 = beta1;
    o->beta2 = beta2;
    o->eps = eps;
    o->weight_decay = weight_decay;
    return o;
}
void ref_adamw_destroy(void* o) { delete static_cast<AdamW*>(o); }
// params[i] (numel[i] doubles) are updated in place from grads[i]; the optimizer keeps m, v by name
int ref_adamw_update(void* o, int64_t n, const char* const* names, double* const* params, const double* const* grads,
                     const int64_t* numel) {
    return guard([&] {
        ParameterSet ps;
        std::map<std::string, Tensor> gs;
        for (int64_t i = 0; i < n; ++i) {
            Tensor w({numel[i]}), g({numel[i]});
            std::memcpy(w.data(), params[i], sizeof(double) * static_cast<size_t>(numel[i]));
            std::memcpy(g.data(), grads[i], sizeof(double) * static_cast<size_t>(numel[i]));
            ps.set(names[i], w);
            gs.emplace(names[i], g);
        }
        static_cast<AdamW*>(o)->update(ps, gs);
        for (int64_t i = 0; i < n; ++i)
            std::memcpy(params[i], ps.at(names[i]).data(), sizeof(double) * static_cast<size_t>(numel[i]));
    });
}

// AdamW::update on a parameter handle's own tensors (the reference FlowTrainer::step's last line,
// flowtrain.cpp:278); grads in ref_params_name order
int ref_adamw_update_params(void* o, void* h, const double* const* grads) {
    return guard([&] {
        auto* hh = static_cast<Handle*>(h);
        std::map<std::string, Tensor> gs;
        for (size_t i = 0; i < hh->names.size(); ++i) {
            const Tensor& w = hh->p.at(hh->names[i]);
            Tensor g(w.shape());
            std::memcpy(g.data(), grads[i], sizeof(double) * static_cast<size_t>(w.numel()));
            gs.emplace(hh->names[i], std::move(g));
        }
        static_cast<AdamW*>(o)->update(hh->p, gs);
    });
}

// ---- post-training (posttrain.cpp) ----
struct RefRecord {  // one post::SampleRecord; cond = first_frame_mask(geom, rows) or no condition
    int64_t dims[3];
    const double* rows;
    int32_t cond;
    const double* text;
    int64_t L;
    double fps;
};

static post::SampleRecord record_of(const RefRecord& r, const dit::DitConfig& cfg) {
    post::SampleRecord s;
    s.geom = geom_of(r.dims, cfg.c_z);
    const int64_t N = s.geom.n(), D = cfg.patch_dim();
    s.rows = Tensor({N, D});
    std::memcpy(s.rows.data(), r.rows, sizeof(double) * static_cast<size_t>(N * D));
    s.mask = r.cond ? flow::first_frame_mask(s.geom, s.rows) : flow::no_condition(N);
    s.text = Tensor({r.L, cfg.text_dim});
    std::memcpy(s.text.data(), r.text, sizeof(double) * static_cast<size_t>(s.text.numel()));
    s.fps = r.fps;
    return s;
}

// post_loss_graph (+ backward when grads_out) on the policy weights `pol` with the frozen `ref`; tag "dpo":
// recs are n pairs as (winner, loser) consecutive records; "kto": n labelled records (desirable flags).
// Draws: make_pair_draws / make_label_draws with Rng(seed).  SFT batch: n_sft samples, shared text / fps.
int ref_post_loss(void* pol, void* ref, const RefCfg* c, const char* tag, double beta, double alpha, double w_d,
                  double w_u, int64_t n, const RefRecord* recs, const int32_t* desirable, int64_t n_sft,
                  const int64_t* sft_dims, const double* const* sft_clean, const double* const* sft_noise,
                  const double* sft_t, const int32_t* sft_cond, const double* sft_text, int64_t sft_L, double sft_fps,
                  uint64_t seed, double* total_out, double* pref_out, double* sft_out, double* grad_norm_out,
                  double* const* grads_out) {
    return guard([&] {
        auto* ph = static_cast<Handle*>(pol);
        auto* rh = static_cast<Handle*>(ref);
        auto cfg = to_cfg(c);
        post::PostTrainConfig pc;
        pc.beta = beta;
        pc.alpha_sft = alpha;
        pc.w_d = w_d;
        pc.w_u = w_u;
        post::PrefBatch batch;
        batch.tag = tag;
        Rng rng(seed);
        std::vector<post::SharedDraw> draws;
        if (batch.tag == "dpo") {
            for (int64_t i = 0; i < n; ++i) {
                post::PreferencePair p;
                p.winner = record_of(recs[2 * i], cfg);
                p.loser = record_of(recs[2 * i + 1], cfg);
                batch.pairs.push_back(std::move(p));
            }
            draws = post::make_pair_draws(batch.pairs, rng);
        } else {
            for (int64_t i = 0; i < n; ++i) {
                post::LabeledSample l;
                l.sample = record_of(recs[i], cfg);
                l.desirable = desirable[i] != 0;
                batch.labels.push_back(std::move(l));
            }
            draws = post::make_label_draws(batch.labels, rng);
        }
        flow::FlowBatch sft;
        sft.text_emb = Tensor({sft_L, cfg.text_dim});
        std::memcpy(sft.text_emb.data(), sft_text, sizeof(double) * static_cast<size_t>(sft.text_emb.numel()));
        sft.fps = sft_fps;
        for (int64_t i = 0; i < n_sft; ++i) {
            flow::FlowSample s;
            s.geom = geom_of(sft_dims + 3 * i, cfg.c_z);
            const int64_t N = s.geom.n(), D = cfg.patch_dim();
            s.clean_rows = Tensor({N, D});
            s.noise = Tensor({N, D});
            std::memcpy(s.clean_rows.data(), sft_clean[i], sizeof(double) * static_cast<size_t>(N * D));
            std::memcpy(s.noise.data(), sft_noise[i], sizeof(double) * static_cast<size_t>(N * D));
            s.t = sft_t[i];
            s.mask = sft_cond[i] ? flow::first_frame_mask(s.geom, s.clean_rows) : flow::no_condition(N);
            sft.samples.push_back(std::move(s));
        }
        Tape t;
        ParamVars pv = register_params(t, ph->p, grads_out != nullptr, "dit.");
        Var pref, sftv;
        Var total = post::post_loss_graph(t, pv, rh->p, cfg, batch, draws, sft, pc, &pref, &sftv);
        *total_out = t.val(total)[0];
        *pref_out = t.val(pref)[0];
        *sft_out = t.val(sftv)[0];
        if (grads_out) {
            t.backward(total);
            auto grads = collect_grads(t, pv);
            *grad_norm_out = flow::grad_norm(grads);
            size_t k = 0;
            for (const auto& nm : ph->names) {
                if (grads_out[k]) {
                    const Tensor& g = grads.at(nm);
                    std::memcpy(grads_out[k], g.data(), sizeof(double) * static_cast<size_t>(g.numel()));
                }
                ++k;
            }
        }
    });
}

// ---- text conditioning (dit.cpp:185-234) ----
int64_t ref_tokenize(const char* prompt, int64_t vocab, int64_t* ids, int64_t cap) {
    dit::DitConfig cfg;
    cfg.text_vocab = vocab;
    std::vector<int64_t> v = dit::tokenize(prompt, cfg);
    for (int64_t k = 0; k < static_cast<int64_t>(v.size()) && k < cap; ++k) ids[k] = v[static_cast<size_t>(k)];
    return static_cast<int64_t>(v.size());
}
// text_embed with text params {text.embed (vocab x D), text.null (1 x D)}; out (L x D); returns L or -1
int64_t ref_text_embed(const int64_t* ids, int64_t n, const double* table, int64_t vocab, const double* null_row,
                       int64_t D, int64_t max_len, double* out, int* truncated) {
    int64_t L = -1;
    guard([&] {
        dit::DitConfig cfg;
        cfg.text_vocab = vocab;
        cfg.text_dim = D;
        cfg.text_max_len = max_len;
        ParameterSet tp;
        Tensor t({vocab, D}), nl({1, D});
        std::memcpy(t.data(), table, sizeof(double) * static_cast<size_t>(vocab * D));
        std::memcpy(nl.data(), null_row, sizeof(double) * static_cast<size_t>(D));
        tp.set("text.embed", std::move(t));
        tp.set("text.null", std::move(nl));
        std::vector<int64_t> v(ids, ids + n);
        dit::TextEmbedding e = dit::text_embed(v, tp, cfg);
        L = e.emb.dim(0);
        std::memcpy(out, e.emb.data(), sizeof(double) * static_cast<size_t>(e.emb.numel()));
        *truncated = e.truncated ? 1 : 0;
    });
    return L;
}

// ---- post-training utilities (posttrain.cpp:51-94, 235-254) ----
int ref_merge_weights(int64_t k, double gamma, double* out) {
    return guard([&] {
        std::vector<real> w = post::merge_weights(k, gamma);
        for (int64_t i = 0; i < k; ++i) out[i] = w[static_cast<size_t>(i)];
    });
}
int ref_anneal_lr(int64_t step, double lr_start, double lr_end, int64_t steps, double* out) {
    return guard([&] {
        post::AnnealConfig c;
        c.lr_start = lr_start;
        c.lr_end = lr_end;
        c.steps = steps;
        *out = post::anneal_lr(step, c);
    });
}
// rdpo_pairs over n records (RefRecord) with the params handle h
int ref_rdpo_pairs(void* h, const RefCfg* c, int64_t n, const RefRecord* recs, int64_t steps, uint64_t seed,
                   double* const* winners, double* const* losers) {
    return guard([&] {
        auto* hh = static_cast<Handle*>(h);
        auto cfg = to_cfg(c);
        std::vector<post::SampleRecord> rs;
        for (int64_t i = 0; i < n; ++i) rs.push_back(record_of(recs[i], cfg));
        std::vector<post::PreferencePair> pairs = post::rdpo_pairs(rs, hh->p, cfg, steps, seed);
        for (int64_t i = 0; i < n; ++i) {
            const auto& p = pairs[static_cast<size_t>(i)];
            std::memcpy(winners[i], p.winner.rows.data(), sizeof(double) * static_cast<size_t>(p.winner.rows.numel()));
            std::memcpy(losers[i], p.loser.rows.data(), sizeof(double) * static_cast<size_t>(p.loser.rows.numel()));
        }
    });
}

// ---- Tape::rope3d (autodiff.cpp:849-898): forward, or the backward's inverse rotation of `x` taken as dL/dy ----
int ref_rope3d(const double* x, int64_t N, int heads, const int* split, const int32_t* coords, double base,
               int inverse, double* out) {
    return guard([&] {
        const std::array<int, 3> sp{split[0], split[1], split[2]};
        const int64_t D = static_cast<int64_t>(heads) * (sp[0] + sp[1] + sp[2]);
        auto co = std::make_shared<std::vector<std::array<int, 3>>>(static_cast<size_t>(N));
        for (int64_t i = 0; i < N; ++i) (*co)[static_cast<size_t>(i)] = {coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]};
        Tensor X({N, D});
        std::memcpy(X.data(), x, sizeof(double) * static_cast<size_t>(N * D));
        Tape t;
        if (!inverse) {
            Var y = t.rope3d(t.constant(X), co, sp, heads, base);
            std::memcpy(out, t.val(y).data(), sizeof(double) * static_cast<size_t>(N * D));
        } else {  // d/dx sum(rope3d(x) * X) = rope_apply_vec(X, -1) accumulated into a zero gradient
            Var xv = t.leaf(Tensor::zeros({N, D}), true);
            Var y = t.rope3d(xv, co, sp, heads, base);
            t.backward(t.sum_all(t.mul(y, t.constant(X))));
            std::memcpy(out, t.grad(xv).data(), sizeof(double) * static_cast<size_t>(N * D));
        }
    });
}

}  // extern "C"
