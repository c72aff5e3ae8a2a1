// Post-training objectives on the device forward (proj/src/posttrain.cpp).
//
// Every preference loss of the reference is a scalar function of per-record masked flow errors
// e_k = flow_error(params, record_k, draw_k) (posttrain.cpp:126-142), so its gradient is
// sum_k (dLoss/de_k) grad e_k.  The device path therefore runs
//   1. forward-only flow errors of the policy and of the frozen reference weights (two contexts),
//   2. the scalar losses and the coefficients dLoss/de_k in fp64 on the host (the closed forms below),
//   3. one weighted fwd+bwd on the policy context over the preference records and the SFT batch
//      (Loss = sum_k w_k e_k), then grad_norm and AdamW on device.
// Step 3 repeats the policy forwards of step 1 (the coefficients need every error first); the forward is
// deterministic, so both passes see bit-identical errors.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "capi_internal.h"
#include "host_rng.h"

namespace {

using mgv::ConfigError;
using mgv::DimensionError;
using mgv::InputError;
using mgv::NumericError;

using HostRng = mgv::HostRng;

double sigmoid(double x) {  // posttrain.cpp:12-16
    if (x >= 0.0) return 1.0 / (1.0 + std::exp(-x));
    const double e = std::exp(x);
    return e / (1.0 + e);
}
double softplus(double x) { return std::max(x, 0.0) + std::log1p(std::exp(-std::fabs(x))); }  // :18

int64_t n_of(const mgv_sample_record& r) { return r.dims[0] * r.dims[1] * r.dims[2]; }

void check_record(const mgv_sample_record& r) {  // posttrain.cpp:20-24 (rows rank / extent; mask checked on staging)
    if (n_of(r) < 1 || !r.rows || !r.coords) throw DimensionError("sample rows do not match the token grid");
    if (!r.text || r.L < 1) throw DimensionError("text embeddings must be (L, text_dim)");
}

void check_pair(const mgv_pref_pair& p) {  // posttrain.cpp:26-32
    check_record(p.winner);
    check_record(p.loser);
    const int64_t n = n_of(p.winner);
    bool same = n == n_of(p.loser);
    if (same) {
        const bool cw = p.winner.conditioned != nullptr, cl = p.loser.conditioned != nullptr;
        for (int64_t i = 0; i < n && same; ++i)
            same = (cw ? p.winner.conditioned[i] != 0 : false) == (cl ? p.loser.conditioned[i] != 0 : false);
    }
    if (!same) throw InputError("pair winner and loser must share conditioning");
}

void validate(const mgv_post_cfg& c) {  // posttrain.cpp:37-49
    if (!(c.beta > 0.0)) throw ConfigError("beta must be > 0");
    if (!(c.alpha_sft >= 0.0)) throw ConfigError("alpha_sft must be >= 0");
    if (!(c.gamma_merge > 0.0) || c.gamma_merge > 1.0) throw ConfigError("gamma_merge must lie in (0, 1]");
    if (!(c.w_d > 0.0) || !(c.w_u > 0.0)) throw ConfigError("kto weights must be > 0");
    if (c.n_interleave < 1 || !c.interleave) throw ConfigError("interleave plan must not be empty");
    for (int64_t i = 0; i < c.n_interleave; ++i) {
        const std::string tag = c.interleave[i] ? c.interleave[i] : "";
        if (tag != "dpo" && tag != "kto") throw ConfigError("unknown interleave tag: " + tag);
    }
}

// SharedDraw (posttrain.hpp:64-68) and make_draw (posttrain.cpp:97-104): t ~ U(0,1] then N x D normals
struct Draw {
    double t = 0.5;
    std::vector<double> noise;
};
Draw make_draw(const mgv_sample_record& r, int64_t D, HostRng& rng) {
    Draw d;
    double u = rng.uniform();
    while (u <= 0.0) u = rng.uniform();
    d.t = u;
    d.noise.resize(static_cast<size_t>(n_of(r) * D));
    for (double& x : d.noise) x = rng.normal();
    return d;
}

mgv_eval_sample eval_of(const mgv_sample_record& r, const Draw& d) {
    mgv_eval_sample e{};
    std::memcpy(e.s.dims, r.dims, sizeof(e.s.dims));
    e.s.coords = r.coords;
    e.s.clean_rows = r.rows;
    e.s.noise = d.noise.data();
    e.s.t = d.t;
    e.s.conditioned = r.conditioned;
    // a record's mask carries its own rows as the condition latents unless given (first_frame_mask, flowtrain.cpp:58)
    e.s.condition_latents = r.conditioned ? (r.condition_latents ? r.condition_latents : r.rows) : nullptr;
    e.text = r.text;
    e.L = r.L;
    e.fps = r.fps;
    return e;
}

struct PrefTerms {
    std::vector<mgv_eval_sample> recs;  // policy records with gradient
    std::vector<double> coef;           // dLoss_pref / de_k
    double loss = 0.0;
};

// dpo_loss_graph (posttrain.cpp:151-169): l_i = softplus(-m_i), m_i = beta((e_th_l - e_th_w) + (e_ref_w - e_ref_l)),
// Loss = mean_i l_i;  dLoss/de_th_w = (beta / P) sigmoid(-m_i) = -dLoss/de_th_l
PrefTerms dpo_terms(mgv::Model& pol, mgv::Model& ref, const mgv_pref_pair* pairs, int64_t n,
                    const std::vector<Draw>& draws, double beta) {
    if (n < 1) throw InputError("empty batch");
    if (static_cast<int64_t>(draws.size()) != n) throw InputError("one shared draw per pair required");
    PrefTerms t;
    for (int64_t i = 0; i < n; ++i) {
        check_pair(pairs[i]);
        t.recs.push_back(eval_of(pairs[i].winner, draws[static_cast<size_t>(i)]));
        t.recs.push_back(eval_of(pairs[i].loser, draws[static_cast<size_t>(i)]));
    }
    std::vector<double> e_th(2 * n), e_ref(2 * n);
    double tmp = 0.0;
    pol.eval_records(2 * n, t.recs.data(), nullptr, e_th.data(), &tmp, nullptr, nullptr);
    ref.eval_records(2 * n, t.recs.data(), nullptr, e_ref.data(), &tmp, nullptr, nullptr);
    double total = 0.0;
    t.coef.resize(static_cast<size_t>(2 * n));
    for (int64_t i = 0; i < n; ++i) {
        const double m = beta * ((e_th[2 * i + 1] - e_th[2 * i]) + (e_ref[2 * i] - e_ref[2 * i + 1]));
        const double li = softplus(-m);
        total = i == 0 ? li : total + li;
        const double g = beta / static_cast<double>(n) * sigmoid(-m);
        t.coef[static_cast<size_t>(2 * i)] = g;
        t.coef[static_cast<size_t>(2 * i + 1)] = -g;
    }
    t.loss = total * (1.0 / static_cast<double>(n));
    return t;
}

// kto_loss_graph (posttrain.cpp:179-222): r_i = beta (e_ref_i - e_th_i), z0 = mean r (detached),
// term_i = w_d sigmoid(-(r_i - z0)) (desirable) or w_u sigmoid(r_i - z0);  Loss = mean_i term_i;
// dLoss/de_th_i = (beta w_d / n) s(1 - s), s = sigmoid(-(r_i - z0))   or   -(beta w_u / n) s(1 - s), s = sigmoid(r_i - z0)
PrefTerms kto_terms(mgv::Model& pol, mgv::Model& ref, const mgv_labeled_sample* labels, int64_t n,
                    const std::vector<Draw>& draws, const mgv_post_cfg& c) {
    if (n < 1) throw InputError("empty batch");
    if (static_cast<int64_t>(draws.size()) != n) throw InputError("one shared draw per sample required");
    PrefTerms t;
    for (int64_t i = 0; i < n; ++i) t.recs.push_back(eval_of(labels[i].sample, draws[static_cast<size_t>(i)]));
    std::vector<double> e_th(n), e_ref(n), r(n);
    double tmp = 0.0;
    pol.eval_records(n, t.recs.data(), nullptr, e_th.data(), &tmp, nullptr, nullptr);
    ref.eval_records(n, t.recs.data(), nullptr, e_ref.data(), &tmp, nullptr, nullptr);
    double z0 = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        r[i] = (-e_th[i] + e_ref[i]) * c.beta;
        z0 += r[i];
    }
    z0 /= static_cast<double>(n);
    double total = 0.0;
    t.coef.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        const double centered = r[i] + -z0;
        double term, g;
        if (labels[i].desirable) {
            const double s = sigmoid(-centered);
            term = s * c.w_d;
            g = c.beta * c.w_d / static_cast<double>(n) * s * (1.0 - s);
        } else {
            const double s = sigmoid(centered);
            term = s * c.w_u;
            g = -c.beta * c.w_u / static_cast<double>(n) * s * (1.0 - s);
        }
        total = i == 0 ? term : total + term;
        t.coef[static_cast<size_t>(i)] = g;
    }
    t.loss = total * (1.0 / static_cast<double>(n));
    return t;
}

std::vector<Draw> pair_draws(const mgv_pref_pair* pairs, int64_t n, int64_t D, HostRng& rng) {  // :106-114
    std::vector<Draw> d;
    for (int64_t i = 0; i < n; ++i) {
        check_pair(pairs[i]);
        d.push_back(make_draw(pairs[i].winner, D, rng));
    }
    return d;
}
std::vector<Draw> label_draws(const mgv_labeled_sample* labels, int64_t n, int64_t D, HostRng& rng) {  // :116-124
    std::vector<Draw> d;
    for (int64_t i = 0; i < n; ++i) {
        check_record(labels[i].sample);
        d.push_back(make_draw(labels[i].sample, D, rng));
    }
    return d;
}

}  // namespace

struct mgv_post_state {
    mgv_ctx* policy = nullptr;
    mgv_ctx* ref = nullptr;
    HostRng rng{0};
    int64_t plan_pos = 0;
    std::string err;
};

extern "C" {

mgv_status mgv_flow_errors(mgv_ctx* ctx, int64_t n, const mgv_eval_sample* recs, double* errs) {
    if (!ctx) return MGV_ERR_INPUT;
    return mgv::guard_into(ctx->err, [&] {
        double loss = 0.0;
        ctx->model->eval_records(n, recs, nullptr, errs, &loss, nullptr, nullptr);
    });
}

mgv_status mgv_flow_step_weighted(mgv_ctx* ctx, int64_t n, const mgv_eval_sample* recs, const double* weights,
                                  double* errs, double* loss, double* grad_norm, double* const* grads_out) {
    if (!ctx) return MGV_ERR_INPUT;
    return mgv::guard_into(ctx->err, [&] {
        if (!weights) throw InputError("null weights");
        ctx->model->eval_records(n, recs, weights, errs, loss, grad_norm, grads_out);
    });
}

mgv_status mgv_post_validate(const mgv_post_cfg* cfg, char* err, int64_t err_cap) {
    std::string msg;
    const mgv_status st = mgv::guard_into(msg, [&] {
        if (!cfg) throw InputError("null config");
        validate(*cfg);
    });
    if (err && err_cap > 0) {
        std::strncpy(err, msg.c_str(), static_cast<size_t>(err_cap - 1));
        err[err_cap - 1] = '\0';
    }
    return st;
}

mgv_status mgv_post_state_create(mgv_ctx* policy, mgv_ctx* ref, double lr, uint64_t seed, mgv_post_state** out) {
    if (!policy || !ref || !out || policy == ref) return MGV_ERR_INPUT;
    *out = nullptr;
    return mgv::guard_into(policy->err, [&] {
        if (policy->model->sorted_params().empty() || ref->model->sorted_params().empty())
            throw InputError("upload the start weights to the policy and the reference contexts first");
        policy->model->set_adamw(lr, 0.9, 0.999, 1e-8, 0.0);  // AdamW(lr) defaults (optim.hpp:12-20)
        auto* st = new mgv_post_state();
        st->policy = policy;
        st->ref = ref;
        st->rng = HostRng(seed);
        *out = st;
    });
}
void mgv_post_state_destroy(mgv_post_state* st) { delete st; }
int64_t mgv_post_plan_pos(const mgv_post_state* st) { return st ? st->plan_pos : 0; }
const char* mgv_post_last_error(const mgv_post_state* st) { return st ? st->err.c_str() : "null state"; }

// post_train_step (posttrain.cpp:292-320) with post_loss_graph (:255-290)
mgv_status mgv_post_train_step(mgv_post_state* st, const mgv_post_cfg* cfg, const char* tag, int64_t n_pairs,
                               const mgv_pref_pair* pairs, int64_t n_labels, const mgv_labeled_sample* labels,
                               int64_t n_sft, const mgv_flow_sample* sft, const double* sft_text, int64_t sft_L,
                               double sft_fps, mgv_post_metrics* out) {
    if (!st) return MGV_ERR_INPUT;
    return mgv::guard_into(st->err, [&] {
        if (!cfg || !tag || !out) throw InputError("null argument");
        validate(*cfg);
        const std::string t(tag);
        const std::string expected = cfg->interleave[st->plan_pos % cfg->n_interleave];
        if (t != expected)
            throw mgv::SchedulingError("batch tag '" + t + "' arrived at a plan position expecting '" + expected + "'");
        mgv::Model& pol = *st->policy->model;
        mgv::Model& ref = *st->ref->model;
        const int64_t D = pol.D();
        const std::vector<Draw> draws =
            t == "dpo" ? pair_draws(pairs, n_pairs, D, st->rng) : label_draws(labels, n_labels, D, st->rng);
        PrefTerms pt = t == "dpo" ? dpo_terms(pol, ref, pairs, n_pairs, draws, cfg->beta)
                                  : kto_terms(pol, ref, labels, n_labels, draws, *cfg);
        if (n_sft < 1 || !sft) throw InputError("empty batch");
        if (!sft_text || sft_L < 1) throw DimensionError("text embeddings must be (L, text_dim)");
        if (!std::isfinite(pt.loss)) throw NumericError("post-training loss is not finite");
        // one weighted fwd+bwd: preference records (coef) + SFT samples (alpha / n_sft), then AdamW
        std::vector<mgv_eval_sample> recs = pt.recs;
        std::vector<double> w = pt.coef;
        for (int64_t j = 0; j < n_sft; ++j) {
            mgv_eval_sample e{};
            e.s = sft[j];
            e.text = sft_text;
            e.L = sft_L;
            e.fps = sft_fps;
            recs.push_back(e);
            w.push_back(cfg->alpha_sft / static_cast<double>(n_sft));
        }
        std::vector<double> errs(recs.size());
        double wl = 0.0, gn = 0.0;
        try {
            pol.eval_records(static_cast<int64_t>(recs.size()), recs.data(), w.data(), errs.data(), &wl, &gn, nullptr);
        } catch (const NumericError&) {
            throw NumericError("post-training loss is not finite");  // the device AdamW step was skipped
        }
        double sft_total = 0.0;  // :281-286
        for (int64_t j = 0; j < n_sft; ++j) {
            const double l = errs[pt.recs.size() + static_cast<size_t>(j)];
            sft_total = j == 0 ? l : sft_total + l;
        }
        sft_total = sft_total * (1.0 / static_cast<double>(n_sft));
        out->preference = pt.loss;
        out->sft = sft_total;
        out->total = pt.loss + sft_total * cfg->alpha_sft;
        out->grad_norm = gn;
        ++st->plan_pos;
    });
}

mgv_status mgv_post_pref_loss(mgv_ctx* policy, mgv_ctx* ref, const mgv_post_cfg* cfg, const char* tag,
                              int64_t n_pairs, const mgv_pref_pair* pairs, int64_t n_labels,
                              const mgv_labeled_sample* labels, uint64_t seed, double* loss) {
    if (!policy || !ref) return MGV_ERR_INPUT;
    return mgv::guard_into(policy->err, [&] {
        if (!cfg || !tag || !loss) throw InputError("null argument");
        const std::string t(tag);
        if (t != "dpo" && t != "kto") throw ConfigError("unknown batch tag: " + t);
        HostRng rng(seed);
        const int64_t D = policy->model->D();
        if (t == "dpo") {
            if (n_pairs < 1) throw InputError("empty batch");  // dpo_loss (:173)
            *loss = dpo_terms(*policy->model, *ref->model, pairs, n_pairs, pair_draws(pairs, n_pairs, D, rng),
                              cfg->beta).loss;
        } else {
            if (n_labels < 1) throw InputError("empty batch");  // kto_loss (:227)
            *loss = kto_terms(*policy->model, *ref->model, labels, n_labels, label_draws(labels, n_labels, D, rng),
                              *cfg).loss;
        }
    });
}

// rdpo_pairs (posttrain.cpp:235-254): per record, reverse-integrate its latents to the noise the model attributes
// to them, then generate the winner forward from that noise and the loser forward from fresh Rng(seed) noise,
// under the record's conditioning, on the device sampler.
mgv_status mgv_rdpo_pairs(mgv_ctx* ctx, int64_t n, const mgv_sample_record* recs, int64_t steps, uint64_t seed,
                          double* const* winners, double* const* losers) {
    if (!ctx) return MGV_ERR_INPUT;
    return mgv::guard_into(ctx->err, [&] {
        if (n < 0 || (n > 0 && (!recs || !winners || !losers))) throw InputError("null argument");
        if (steps < 1) throw InputError("steps must be >= 1");  // flowtrain.cpp:137
        mgv::Model& m = *ctx->model;
        const int64_t D = m.D();
        HostRng rng(seed);
        for (int64_t k = 0; k < n; ++k) {
            const mgv_sample_record& r = recs[k];
            check_record(r);
            const int64_t N = n_of(r);
            const double* cl = r.conditioned ? (r.condition_latents ? r.condition_latents : r.rows) : nullptr;
            std::vector<double> noise_hat(static_cast<size_t>(N * D)), fresh(static_cast<size_t>(N * D));
            m.sample_rows(r.rows, N, r.coords, r.dims, r.text, r.L, r.conditioned, cl, steps, +1, r.fps,
                          noise_hat.data());  // reverse_sample_rows
            m.sample_rows(noise_hat.data(), N, r.coords, r.dims, r.text, r.L, r.conditioned, cl, steps, -1, r.fps,
                          winners[k]);  // forward_sample_rows
            for (double& x : fresh) x = rng.normal();
            m.sample_rows(fresh.data(), N, r.coords, r.dims, r.text, r.L, r.conditioned, cl, steps, -1, r.fps,
                          losers[k]);
        }
    });
}

// merge_weights / anneal_lr (posttrain.cpp:51-94)
mgv_status mgv_merge_weights(int64_t k, double gamma, double* out) {
    std::string msg;
    return mgv::guard_into(msg, [&] {
        if (k < 1) throw InputError("need at least one checkpoint");
        if (!(gamma > 0.0) || gamma > 1.0) throw ConfigError("gamma must lie in (0, 1]");
        if (!out) throw InputError("null output");
        double total = 0.0;
        for (int64_t i = 0; i < k; ++i) {
            out[i] = std::pow(gamma, static_cast<double>(k - 1 - i));
            total += out[i];
        }
        for (int64_t i = 0; i < k; ++i) out[i] /= total;
    });
}
mgv_status mgv_anneal_lr(int64_t step, double lr_start, double lr_end, int64_t steps, double* out) {
    std::string msg;
    return mgv::guard_into(msg, [&] {
        if (steps < 2) throw ConfigError("anneal horizon needs at least two steps");
        if (!(lr_start > 0.0) || !(lr_end >= 0.0) || lr_end > lr_start)
            throw ConfigError("anneal must decay from lr_start to lr_end");
        if (step < 0) throw InputError("anneal step must be >= 0");
        if (!out) throw InputError("null output");
        if (step >= steps - 1) {
            *out = lr_end;
        } else if (step == 0) {
            *out = lr_start;
        } else {
            const double frac = static_cast<double>(step) / static_cast<double>(steps - 1);
            *out = lr_end + (lr_start - lr_end) * 0.5 * (1.0 + std::cos(M_PI * frac));
        }
    });
}

double mgv_dpo_from_errors(double e_th_w, double e_th_l, double e_ref_w, double e_ref_l, double beta) {
    const double margin = beta * ((e_ref_w - e_th_w) - (e_ref_l - e_th_l));  // posttrain.cpp:144-147
    return softplus(-margin);
}

mgv_status mgv_kto_from_rewards(int64_t n, const double* rewards, const uint8_t* desirable, double w_d, double w_u,
                                const double* z0_override, double* out) {
    std::string msg;
    return mgv::guard_into(msg, [&] {  // posttrain.cpp:184-204
        if (n < 1 || !rewards) throw InputError("empty batch");
        if (!desirable || !out) throw InputError("one desirability flag per reward required");
        double z0 = 0.0;
        if (z0_override) {
            z0 = *z0_override;
        } else {
            for (int64_t i = 0; i < n; ++i) z0 += rewards[i];
            z0 /= static_cast<double>(n);
        }
        double total = 0.0;
        for (int64_t i = 0; i < n; ++i)
            total += desirable[i] ? w_d * (1.0 - sigmoid(rewards[i] - z0)) : w_u * (1.0 - sigmoid(z0 - rewards[i]));
        *out = total / static_cast<double>(n);
    });
}

}  // extern "C"
