// Drop-in binding of the B200 library (include/mugv_b200.h) into the reference's C++ API (proj/include/mugv).
//
// Link this translation unit ahead of the reference library, with the replaced definitions in the reference's
// dit.o weakened (shim/Makefile: objcopy --weaken-symbol), and every caller of the hot path runs on the GPU:
//
//   mugv::dit::velocity_rows_graph (dit.hpp:124-127, dit.cpp:320-334)
//       ONE tape node through mugv::TapeOps (the friend autodiff.hpp:134 leaves undefined): the value (and the
//       reference's taps) from the device forward, and a backward closure that runs the device VJP and adds the
//       dit.* parameter gradients into the tape.  So the reference's own FlowTrainer::step (flowtrain.cpp:257-282),
//       posttrain flow errors (posttrain.cpp:126-142, 284), expansion::verify_preservation (expansion.cpp:267-272)
//       and predict_velocity (dit.cpp:388-396) run the block on the B200 unchanged, with the reference's tape,
//       loss, grad norm and AdamW around it.
//   mugv::dit::dit_forward / dit_forward_batch (dit.hpp:94-100, dit.cpp:361-386)
//       the value API on the device (mgv_dit_forward).
//   mugv::dit::predict_velocity (dit.hpp:104-106): mgv_predict_velocity.
//
// Contexts: one device context per (thread, precision); the dit.* weights are cached on it and re-uploaded only
// when the content fingerprint of the ParameterSet / tape leaves changes (the API re-passes them on every call).
// A trainer's weights change every step, so each step uploads them once (fp64 -> fp32 masters).  Errors come back
// as the reference's exception types (errors.hpp).  Precision: MUGV_B200_PRECISION = fp32 (default; the parity
// mode, <= 1e-4 of the fp64 reference) or bf16; device: MUGV_B200_DEVICE (default 0).
//
// mugv::b200::DeviceFlowTrainer: FlowTrainer's interface (ctor, step, params, optimizer hyper-parameters) with the
// whole step -- interpolation, masks, fwd, bwd, grad norm and AdamW -- on the device (mgv_flow_step), one context
// per trainer; params() downloads the device weights.
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "mugv/dit.hpp"
#include "mugv/errors.hpp"
#include "mugv/flowtrain.hpp"
#include "mugv/graph.hpp"
#include "mugv_b200.h"
#include "mugv_b200_shim.hpp"

namespace mugv {

// The friend of Tape (autodiff.hpp:134): the only way a node computed outside the tape can join it.
struct TapeOps {
    static Var push(Tape& t, Tensor val, bool requires_grad, std::function<void(Tape&, Var)> back) {
        return t.push(std::move(val), requires_grad, std::move(back));
    }
    static bool needs(const Tape& t, Var v) { return t.needs(v); }
    static Tensor& gbuf(Tape& t, Var v) { return t.gbuf(v); }
    static const Tensor& node_grad(const Tape& t, Var v) { return t.nodes_[t.check(v)].grad; }
};

namespace b200 {
namespace {

[[noreturn]] void rethrow(mgv_status st, const std::string& what) {
    switch (st) {
        case MGV_ERR_DIMENSION: throw DimensionError(what);
        case MGV_ERR_CONFIG: throw ConfigError(what);
        case MGV_ERR_INPUT: throw InputError(what);
        case MGV_ERR_NUMERIC: throw NumericError(what);
        default: throw std::runtime_error("mugv_b200: " + what);
    }
}

void check(mgv_ctx* ctx, mgv_status st) {
    if (st != MGV_OK) rethrow(st, ctx ? mgv_last_error(ctx) : "no device context");
}

int env_precision() {
    const char* e = std::getenv("MUGV_B200_PRECISION");
    return e && std::string(e) == "bf16" ? MGV_PREC_BF16 : MGV_PREC_FP32;
}
int env_device() {
    const char* e = std::getenv("MUGV_B200_DEVICE");
    return e ? std::atoi(e) : 0;
}

mgv_dit_cfg to_c(const dit::DitConfig& c) {
    mgv_dit_cfg g{};
    g.depth = c.depth;
    g.hidden = c.hidden;
    g.heads = c.heads;
    g.text_dim = c.text_dim;
    g.c_z = c.c_z;
    for (int i = 0; i < 3; ++i) g.rope_split[i] = c.rope_split[static_cast<size_t>(i)];
    g.text_vocab = c.text_vocab;
    g.text_max_len = c.text_max_len;
    return g;
}

// FNV-1a over the config, names, shapes and raw values
struct Fingerprint {
    uint64_t h = 1469598103934665603ull;
    void bytes(const void* p, size_t n) {
        const auto* b = static_cast<const unsigned char*>(p);
        for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    }
    void words(const double* p, int64_t n) {  // 8 bytes per step: hashing 10B-scale weights stays cheap
        for (int64_t i = 0; i < n; ++i) {
            uint64_t w;
            std::memcpy(&w, p + i, 8);
            h = (h ^ w) * 1099511628211ull;
            h ^= h >> 29;
        }
    }
};

struct Weights {  // a dit.* parameter set as parallel arrays
    std::vector<std::string> names;
    std::vector<const double*> data;
    std::vector<int64_t> numel;
    uint64_t fingerprint(const dit::DitConfig& cfg) const {
        Fingerprint f;
        const mgv_dit_cfg c = to_c(cfg);
        f.bytes(&c, sizeof(c));
        for (size_t i = 0; i < names.size(); ++i) {
            f.bytes(names[i].data(), names[i].size());
            f.bytes(&numel[i], sizeof(int64_t));
            f.words(data[i], numel[i]);
        }
        return f.h;
    }
};

Weights from_params(const ParameterSet& p) {
    Weights w;
    for (const std::string& n : p.names()) {
        if (n.rfind("dit.", 0) != 0) continue;  // register_params(..., "dit.") (dit.cpp:366, 392)
        const Tensor& t = p.at(n);
        w.names.push_back(n);
        w.data.push_back(t.data());
        w.numel.push_back(t.numel());
    }
    return w;
}

Weights from_tape(const Tape& t, const ParamVars& pv) {
    Weights w;
    for (const auto& [n, v] : pv.all()) {
        if (n.rfind("dit.", 0) != 0) continue;
        const Tensor& x = t.val(v);
        w.names.push_back(n);
        w.data.push_back(x.data());
        w.numel.push_back(x.numel());
    }
    return w;
}

// One device context per (thread, precision) with its weight cache (the reference API is re-entrant and callers
// are single-threaded per object)
class Device {
public:
    explicit Device(int precision) {
        if (mgv_ctx_create(env_device(), precision, &ctx_) != MGV_OK)
            throw std::runtime_error("mugv_b200: no CUDA device for the drop-in (mgv_ctx_create failed)");
    }
    ~Device() { mgv_ctx_destroy(ctx_); }
    mgv_ctx* ctx() const { return ctx_; }

    // make the context hold these weights (no-op when the fingerprint matches the resident set)
    void ensure(const Weights& w, const dit::DitConfig& cfg) {
        const uint64_t fp = w.fingerprint(cfg);
        if (have_ && fp == fp_) return;
        std::vector<const char*> nm;
        for (const auto& s : w.names) nm.push_back(s.c_str());
        const mgv_dit_cfg c = to_c(cfg);
        check(ctx_, mgv_params_upload(ctx_, &c, static_cast<int64_t>(nm.size()), nm.data(), w.data.data(),
                                      w.numel.data()));
        names_.clear();
        for (int64_t i = 0; i < mgv_param_count(ctx_); ++i) names_.emplace_back(mgv_param_name(ctx_, i));
        fp_ = fp;
        have_ = true;
    }
    const std::vector<std::string>& names() const { return names_; }

private:
    mgv_ctx* ctx_ = nullptr;
    bool have_ = false;
    uint64_t fp_ = 0;
    std::vector<std::string> names_;
};

Device& device() {
    thread_local std::map<int, std::unique_ptr<Device>> devs;
    const int p = env_precision();
    auto& d = devs[p];
    if (!d) d = std::make_unique<Device>(p);
    return *d;
}

std::vector<int32_t> coords_of(const dit::TokenGrid& g, int64_t N) {
    if (!g.coords || static_cast<int64_t>(g.coords->size()) != N)
        throw DimensionError("token coords do not match the rows");
    std::vector<int32_t> c(static_cast<size_t>(3 * N));
    for (int64_t i = 0; i < N; ++i)
        for (int k = 0; k < 3; ++k) c[static_cast<size_t>(3 * i + k)] = (*g.coords)[static_cast<size_t>(i)][k];
    return c;
}

}  // namespace
}  // namespace b200

namespace dit {

Var velocity_rows_graph(Tape& t, Var rows, const TokenGrid& geom, Var text, const Tensor& timesteps, real fps,
                        const ParamVars& pv, const DitConfig& cfg, std::vector<Var>* taps) {
    using namespace b200;
    const Tensor& rv = t.val(rows);  // the reference's own shape checks first (dit.cpp:322-325)
    if (rv.rank() != 2 || rv.dim(1) != cfg.patch_dim())
        throw DimensionError("latent rows must be (N, 4*c_z), got " + rv.shape_str());
    if (timesteps.rank() != 1 || timesteps.dim(0) != rv.dim(0)) throw DimensionError("need one timestep per token");
    if (TapeOps::needs(t, rows) || TapeOps::needs(t, text))
        throw InputError("velocity_rows_graph on the device: rows and text must be constants of the graph");
    const Tensor& tx = t.val(text);
    if (tx.rank() != 2 || tx.dim(1) != cfg.text_dim) throw DimensionError("text embeddings must be (L, text_dim)");
    const int64_t N = rv.dim(0), L = tx.dim(0), H = cfg.hidden, D = cfg.patch_dim();
    Device& dev = device();
    const Weights w = from_tape(t, pv);
    dev.ensure(w, cfg);
    auto coords = std::make_shared<std::vector<int32_t>>(coords_of(geom, N));
    const int64_t dims[3] = {geom.dims[0], geom.dims[1], geom.dims[2]};
    Tensor V({N, D});
    std::vector<Tensor> tap_vals;
    std::vector<double*> tap_ptrs;
    if (taps) {
        for (int64_t i = 0; i < cfg.depth + 2; ++i) tap_vals.emplace_back(std::vector<int64_t>{N, H});
        tap_vals.emplace_back(std::vector<int64_t>{N, D});
        for (Tensor& x : tap_vals) tap_ptrs.push_back(x.data());
    }
    check(dev.ctx(), mgv_velocity_graph(dev.ctx(), rv.data(), N, coords->data(), dims, tx.data(), L, timesteps.data(),
                                        fps, V.data(), taps ? tap_ptrs.data() : nullptr, nullptr, nullptr));
    bool req = false;
    for (const auto& [n, v] : pv.all())
        if (n.rfind("dit.", 0) == 0) req = req || TapeOps::needs(t, v);
    std::map<std::string, Var> vars;
    for (const auto& [n, v] : pv.all())
        if (n.rfind("dit.", 0) == 0) vars[n] = v;
    // backward closure: the device VJP of this node, added into the parameter leaves' gradients
    Var out = TapeOps::push(
        t, std::move(V), req,
        [rows, text, timesteps, fps, cfg, coords, dims = std::array<int64_t, 3>{dims[0], dims[1], dims[2]}, N, L,
         vars](Tape& tt, Var self) {
            Device& d = device();
            ParamVars pv2;
            for (const auto& [n, v] : vars) pv2.put(n, v);
            d.ensure(from_tape(tt, pv2), cfg);  // the weights this node was built on (still on the tape)
            const Tensor& dV = TapeOps::node_grad(tt, self);
            std::vector<Tensor> g;
            std::vector<double*> gp;
            for (const std::string& n : d.names()) {
                auto it = vars.find(n);
                const bool want = it != vars.end() && TapeOps::needs(tt, it->second);
                g.emplace_back(want ? tt.val(it->second).shape() : std::vector<int64_t>{0});
                gp.push_back(want ? g.back().data() : nullptr);
            }
            check(d.ctx(), mgv_velocity_graph(d.ctx(), tt.val(rows).data(), N, coords->data(), dims.data(),
                                              tt.val(text).data(), L, timesteps.data(), fps, nullptr, nullptr,
                                              dV.data(), gp.data()));
            for (size_t k = 0; k < d.names().size(); ++k) {
                if (!gp[k]) continue;
                Tensor& acc = TapeOps::gbuf(tt, vars.at(d.names()[k]));
                for (int64_t e = 0; e < acc.numel(); ++e) acc[e] += g[k][e];
            }
        });
    if (taps) {  // patch embedding, block outputs, final projection, velocity (dit.cpp:326-332)
        for (size_t i = 0; i + 1 < tap_vals.size(); ++i) taps->push_back(t.constant(std::move(tap_vals[i])));
        taps->push_back(out);
    }
    return out;
}

TokenGrid dit_forward(const TokenGrid& tokens, const Tensor& text_emb, const GlobalSignals& signals,
                      const ParameterSet& params, const DitConfig& cfg) {
    using namespace b200;
    validate(cfg);
    if (signals.timestep.rank() != 1 || signals.timestep.dim(0) != tokens.tokens.dim(0))
        throw DimensionError("need one timestep per token");
    const Tensor& tk = tokens.tokens;
    if (tk.rank() != 2 || tk.dim(1) != cfg.hidden) throw DimensionError("tokens must be (N, hidden)");
    if (text_emb.rank() != 2 || text_emb.dim(1) != cfg.text_dim)
        throw DimensionError("text embeddings must be (L, text_dim)");
    const int64_t N = tk.dim(0);
    Device& dev = device();
    dev.ensure(from_params(params), cfg);
    const std::vector<int32_t> co = coords_of(tokens, N);
    const int64_t dims[3] = {tokens.dims[0], tokens.dims[1], tokens.dims[2]};
    TokenGrid out;
    out.tokens = Tensor({N, cfg.hidden});
    check(dev.ctx(), mgv_dit_forward(dev.ctx(), tk.data(), N, co.data(), dims, text_emb.data(), text_emb.dim(0),
                                     signals.timestep.data(), signals.fps, out.tokens.data()));
    out.coords = tokens.coords;
    out.dims = tokens.dims;
    return out;
}

std::vector<TokenGrid> dit_forward_batch(const std::vector<TokenGrid>& batch, const Tensor& text_emb,
                                         const std::vector<GlobalSignals>& signals, const ParameterSet& params,
                                         const DitConfig& cfg) {
    if (batch.size() != signals.size()) throw DimensionError("one GlobalSignals entry per sample");
    std::vector<TokenGrid> out;
    out.reserve(batch.size());
    for (size_t i = 0; i < batch.size(); ++i) out.push_back(dit_forward(batch[i], text_emb, signals[i], params, cfg));
    return out;
}

Tensor predict_velocity(const Tensor& rows, const TokenGrid& geom, const Tensor& text_emb, const Tensor& timesteps,
                        real fps, const ParameterSet& params, const DitConfig& cfg) {
    using namespace b200;
    validate(cfg);
    if (rows.rank() != 2 || rows.dim(1) != cfg.patch_dim())
        throw DimensionError("latent rows must be (N, 4*c_z), got " + rows.shape_str());
    if (timesteps.rank() != 1 || timesteps.dim(0) != rows.dim(0)) throw DimensionError("need one timestep per token");
    if (text_emb.rank() != 2 || text_emb.dim(1) != cfg.text_dim)
        throw DimensionError("text embeddings must be (L, text_dim)");
    const int64_t N = rows.dim(0);
    Device& dev = device();
    dev.ensure(from_params(params), cfg);
    const std::vector<int32_t> co = coords_of(geom, N);
    const int64_t dims[3] = {geom.dims[0], geom.dims[1], geom.dims[2]};
    Tensor out({N, cfg.patch_dim()});
    check(dev.ctx(), mgv_predict_velocity(dev.ctx(), rows.data(), N, co.data(), dims, text_emb.data(), text_emb.dim(0),
                                          timesteps.data(), fps, out.data()));
    return out;
}

}  // namespace dit

// ------------------------------------------------------------------ the whole step on the device
namespace b200 {

struct DeviceFlowTrainer::Impl {
    mgv_ctx* ctx = nullptr;
    dit::DitConfig cfg;
    ParameterSet params;  // host mirror, refreshed lazily by params()
    bool stale = false;
    ~Impl() { mgv_ctx_destroy(ctx); }
};

DeviceFlowTrainer::DeviceFlowTrainer(ParameterSet dit_params, dit::DitConfig cfg, real lr, int precision)
    : impl_(std::make_unique<Impl>()) {
    dit::validate(cfg);  // FlowTrainer::FlowTrainer (flowtrain.cpp:252-255)
    impl_->cfg = cfg;
    impl_->params = std::move(dit_params);
    if (mgv_ctx_create(env_device(), precision < 0 ? env_precision() : precision, &impl_->ctx) != MGV_OK)
        throw std::runtime_error("mugv_b200: no CUDA device (mgv_ctx_create failed)");
    AdamW defaults(lr);  // optim.hpp:14-18 hyper-parameters
    check(impl_->ctx, mgv_ctx_set_adamw(impl_->ctx, defaults.lr, defaults.beta1, defaults.beta2, defaults.eps,
                                        defaults.weight_decay));
    const Weights w = from_params(impl_->params);
    std::vector<const char*> nm;
    for (const auto& s : w.names) nm.push_back(s.c_str());
    const mgv_dit_cfg c = to_c(cfg);
    check(impl_->ctx, mgv_params_upload(impl_->ctx, &c, static_cast<int64_t>(nm.size()), nm.data(), w.data.data(),
                                        w.numel.data()));  // once: the AdamW moments live on the device
}

DeviceFlowTrainer::~DeviceFlowTrainer() = default;

flow::StepMetrics DeviceFlowTrainer::step(const flow::FlowBatch& batch) {
    if (batch.samples.empty()) throw InputError("empty batch");  // flowtrain.cpp:258
    const int64_t D = impl_->cfg.patch_dim();
    std::vector<mgv_flow_sample> ss(batch.samples.size());
    std::vector<std::vector<int32_t>> coords(batch.samples.size());
    for (size_t i = 0; i < batch.samples.size(); ++i) {
        const flow::FlowSample& s = batch.samples[i];
        const int64_t N = s.geom.n();
        if (s.clean_rows.rank() != 2 || s.clean_rows.dim(0) != N || s.clean_rows.dim(1) != D || !s.noise.same_shape(s.clean_rows))
            throw DimensionError("sample rows must be (N, 4*c_z)");
        coords[i] = coords_of(s.geom, N);
        mgv_flow_sample& c = ss[i];
        for (int k = 0; k < 3; ++k) c.dims[k] = s.geom.dims[static_cast<size_t>(k)];
        c.coords = coords[i].data();
        c.clean_rows = s.clean_rows.data();
        c.noise = s.noise.data();
        c.t = s.t;
        if (s.mask.any()) {
            if (static_cast<int64_t>(s.mask.conditioned.size()) != N)
                throw DimensionError("condition mask does not match the token grid");
            c.conditioned = s.mask.conditioned.data();
            if (s.mask.condition_latents.rank() != 2 || s.mask.condition_latents.dim(0) != N ||
                s.mask.condition_latents.dim(1) != D)
                throw InputError("condition mask lacks clean latents for its conditioned tokens");
            c.condition_latents = s.mask.condition_latents.data();
        }
    }
    const Tensor& tx = batch.text_emb;
    if (tx.rank() != 2 || tx.dim(1) != impl_->cfg.text_dim) throw DimensionError("text embeddings must be (L, text_dim)");
    flow::StepMetrics m;
    check(impl_->ctx, mgv_flow_step(impl_->ctx, static_cast<int64_t>(ss.size()), ss.data(), tx.data(), tx.dim(0),
                                    batch.fps, &m.loss, &m.grad_norm, nullptr, nullptr));
    impl_->stale = true;
    return m;
}

const ParameterSet& DeviceFlowTrainer::params() {
    if (impl_->stale) {  // the device fp32 masters, widened
        for (int64_t i = 0; i < mgv_param_count(impl_->ctx); ++i) {
            Tensor& t = impl_->params.at(mgv_param_name(impl_->ctx, i));
            check(impl_->ctx, mgv_param_download(impl_->ctx, i, t.data()));
        }
        impl_->stale = false;
    }
    return impl_->params;
}

int64_t DeviceFlowTrainer::step_count() const { return mgv_adamw_steps(impl_->ctx); }
const dit::DitConfig& DeviceFlowTrainer::config() const { return impl_->cfg; }

}  // namespace b200
}  // namespace mugv
