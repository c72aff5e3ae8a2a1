// C++ runtime of the DiT hot path: device weight cache, workspace arena, and
// the forward / backward orchestration of velocity_rows_graph + flow loss
// (proj/src/dit.cpp:267-334, proj/src/flowtrain.cpp:257-289).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mugv_b200.h"

namespace mgv {

// Errors mirroring the reference taxonomy (errors.hpp); mapped to mgv_status at the C ABI.
struct DimensionError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct InputError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NumericError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NcclError : std::runtime_error { using std::runtime_error::runtime_error; };

struct Cfg {
    int64_t depth = 0, hidden = 0, heads = 0, text_dim = 0, c_z = 0;
    int rope[3] = {0, 0, 0};
    int64_t H() const { return hidden; }
    int64_t hd() const { return hidden / heads; }
    int64_t D() const { return 4 * c_z; }
};
void validate_cfg(const Cfg& c);
// bytes one rank allocates for a step: out = {parameters, gradients, AdamW moments, workspace, exchange arena}
// train: 0 forward only, 1 training step, 3 training step with per-block activation recompute
void plan_rank_bytes(const Cfg& c, bool bf16, int tp, int64_t N, int64_t L, int n_u, int train, int64_t out[5]);

struct DevParam {
    std::string name;
    std::vector<int64_t> shape;
    int64_t numel = 0;              // elements held by this process (a real TP rank: its shard of sharded params)
    int64_t numel_full = 0;         // elements of the reference tensor
    int64_t slot_numel = 0;         // elements of one TP rank's slot (numel_full / P for sharded params)
    int shard = 0;                  // 0 replicated, 1 row-parallel (rank-major rows), 2 column-parallel (compact)
    float* f32 = nullptr;           // master copy (all params)
    __nv_bfloat16* bf = nullptr;    // tensor-core operand copy (matrices, bf16 mode)
    float* grad = nullptr;          // slice of the contiguous gradient buffer
    int64_t grad_off = 0;
};

// Device sample (all pointers device-resident).
struct DevSample {
    int64_t N = 0;
    int64_t dims[3] = {0, 0, 0};
    const int32_t* coords = nullptr;
    const double* clean = nullptr;
    const double* noise = nullptr;
    double t = 0.0;
    const uint8_t* cond = nullptr;     // N condition flags (ConditionMask::conditioned, flowtrain.hpp:32-41) or null
    const double* cond_lat = nullptr;  // N x D condition latents (read at conditioned rows only) or null (= clean)
};

// Per-sample overrides of a flow step (post-training, posttrain.cpp:126-233): every sample may carry its own
// text and fps and a loss weight, and the step may be forward-only (flow errors, no gradients).
struct StepExtra {
    const double* const* text_dev = nullptr;  // per-sample device text (L[k] x text_dim); null: the step's text
    const int64_t* L = nullptr;
    const double* fps = nullptr;
    const double* weight = nullptr;  // dLoss/d l_k; null: 1 / global batch (FlowTrainer::step)
    bool backward = true;            // false: forward only, no gradients, no optimizer update
    double* errs = nullptr;          // host out: each sample's masked flow loss l_k (flowtrain.cpp:22-38)
};

class Arena {
public:
    ~Arena();
    void reserve(size_t bytes);
    void reset() { off_ = 0; }
    template <class T>
    T* take(int64_t n) {
        size_t bytes = (sizeof(T) * static_cast<size_t>(n) + 255) & ~size_t(255);
        if (off_ + bytes > cap_) throw std::runtime_error("workspace arena overflow");
        T* p = reinterpret_cast<T*>(base_ + off_);
        off_ += bytes;
        return p;
    }
    size_t used() const { return off_; }
    size_t cap() const { return cap_; }

private:
    char* base_ = nullptr;
    size_t cap_ = 0, off_ = 0;
};

// Optional per-phase device timing (CUDA events on the launching stream), used by the
// benchmark for the roofline figures.  Off by default; no host syncs when on.
class Prof {
public:
    struct Stat {
        double ms = 0.0;
        int64_t n = 0;
        double work = 0.0;  // algorithmic FLOPs of the phase's launches (GEMM phase)
    };
    bool on = false;
    std::map<std::string, Stat> stats;
    void begin_step() { pend_.clear(); }
    void begin(const char* name, cudaStream_t s, double work = 0.0);
    void end(cudaStream_t s);
    void end_step();  // after the stream was synchronised
    ~Prof();

private:
    struct Pend {
        std::string name;
        cudaEvent_t a, b;
        double work;
    };
    cudaEvent_t get();
    std::vector<Pend> pend_;
    std::vector<cudaEvent_t> pool_, used_;
};

// Routes the bf16 GEMM launches of one step into `p` as the "gemm" phase while alive (profiling only).
struct GemmProfGuard {
    explicit GemmProfGuard(Prof& p);
    ~GemmProfGuard();
};

class Model {
public:
    Model(int device, bool bf16);
    ~Model();

    void set_stream(cudaStream_t s) { stream_ = s; }
    void set_dp(int rank, int world, const uint8_t id[128]);
    // Megatron tensor parallelism over `size` ranks.  id == nullptr: all `size` ranks are
    // emulated in this process (sequentially, partial sums accumulated in place of the all-reduce);
    // otherwise this process is TP rank `rank` of an NCCL communicator.  Must precede upload().
    void set_tp(int size, int rank, const uint8_t* id);
    int tp_size() const { return tp_; }
    // varlen packing of multi-sample flow steps (flow_step_packed); off: samples run one after another
    void set_varlen(bool on) { varlen_ = on; }
    void set_recompute(bool on) { recompute_ = on; }
    bool varlen() const { return varlen_; }
    void memory_bytes(int64_t out[5]) const;  // this context's allocations, same categories as plan_rank_bytes
    // AdamW::update after every flow step (optim.cpp:7-24, flowtrain.cpp:278); lr <= 0 disables
    void set_adamw(double lr, double beta1, double beta2, double eps, double weight_decay);
    int64_t adamw_steps() const { return adam_.step; }
    // parameter i (sorted-name order) in the reference layout, fp64
    void download_param(int64_t i, double* out);

    void upload(const Cfg& cfg, int64_t n, const char* const* names, const double* const* data,
                const int64_t* numel) {
        upload(cfg, n, names, reinterpret_cast<const void* const*>(data), nullptr, numel);
    }
    // is_f32[i] != 0: data[i] is float (a checkpoint's f32 payload, uploaded bit-exactly); nullptr = all fp64
    void upload(const Cfg& cfg, int64_t n, const char* const* names, const void* const* data, const uint8_t* is_f32,
                const int64_t* numel);
    const std::vector<DevParam*>& sorted_params() const { return sorted_; }

    // Host-buffer entry points (the C ABI).
    void predict_velocity(const double* rows, int64_t N, const int32_t* coords, const int64_t dims[3],
                          const double* text, int64_t L, const double* tau, double fps, double* out);
    void dit_forward(const double* tokens, int64_t N, const int32_t* coords, const int64_t dims[3],
                     const double* text, int64_t L, const double* tau, double fps, double* out);
    // The tape-level builder velocity_rows_graph (dit.cpp:320-334) as one device node: forward with the reference's
    // taps (patch embedding, each block's residual output, the final normed projection, the velocity; any output
    // pointer may be null) and, when dV is given, the vector-Jacobian product: gradients of sum(dV * V) w.r.t.
    // every dit.* parameter (sorted-name order, overwritten) -- the node's backward closure.
    void velocity_graph(const double* rows, int64_t N, const int32_t* coords, const int64_t dims[3],
                        const double* text, int64_t L, const double* tau, double fps, double* V_out,
                        double* const* taps_out, const double* dV, double* const* grads_out);
    // dit::patchify / unpatchify / global_embed (dit.hpp:83-90): the projections at either end of the block
    // stack and the timestep/fps embedding, from the device weights (fp32 masters, IEEE-fp32 GEMMs)
    void patchify(const double* grid, int64_t U, int64_t h, int64_t w, int64_t C, double* tokens, int32_t* coords);
    void unpatchify(const double* tokens, int64_t N, const int32_t* coords, const int64_t dims[3], double* grid);
    void global_embed_host(const double* tau, int64_t N, double fps, double* g, double* block_scales);
    // forward_sample_rows / reverse_sample_rows (flowtrain.cpp:135-172): `steps` Euler steps of the
    // probability-flow ODE on device (direction -1: t 1 -> 0, x -= dt v; +1: t 0 -> 1, x += dt v),
    // conditioned rows re-imposed after every step.  cond / cond_latents may be null.
    void sample_rows(const double* x_start, int64_t N, const int32_t* coords, const int64_t dims[3],
                     const double* text, int64_t L, const uint8_t* cond, const double* cond_latents, int64_t steps,
                     int direction, double fps, double* out);
    void flow_step(int64_t n, const mgv_flow_sample* samples, const double* text, int64_t L, double fps,
                   double* loss, double* grad_norm, double* const* grads_out, double* const* v_out);
    // Post-training evaluations (posttrain.cpp:126-142): per-record text / fps; errs[k] = l_k.  weights null:
    // forward only (flow_error); else one fwd+bwd with Loss = sum_k w_k l_k, grads = sum_k w_k dl_k (then
    // grad_norm and, when enabled, AdamW), loss = sum_k w_k l_k.
    void eval_records(int64_t n, const mgv_eval_sample* recs, const double* weights, double* errs, double* loss,
                      double* grad_norm, double* const* grads_out);
    // Device-resident inputs (benchmark `value` path): no host<->device traffic except the two scalars.
    void flow_step_dev(int64_t n, const DevSample* samples, const double* text_dev, int64_t L, double fps,
                       double* loss, double* grad_norm, double* const* v_dev = nullptr,
                       const StepExtra* ex = nullptr);

    double last_step_ms() const { return last_ms_; }
    int64_t last_step_launches() const { return last_launches_; }
    Prof& prof() { return prof_; }
    bool bf16() const { return bf16_; }
    int64_t D() const { return cfg_.D(); }
    cudaStream_t stream() const { return stream_; }

private:
    template <class T>
    void flow_step_impl(int64_t n, const DevSample* samples, const double* text_dev, int64_t L, double fps,
                        double* loss, double* grad_norm, double* const* v_dev, const StepExtra* ex);
    template <class T>
    void flow_step_packed(int64_t n, const DevSample* samples, const double* text_dev, int64_t L, double fps,
                          double* loss, double* grad_norm, double* const* v_dev);
    void adamw_step(cudaStream_t s);
    void stage_samples(int64_t n, const mgv_flow_sample* samples, std::vector<DevSample>& ds,
                       std::vector<void*>& allocs);
    template <class Alloc>
    void download_grads(double* const* grads_out, Alloc&& dalloc);
    template <class T>
    void forward_sample(const DevSample& s, const void* rows_in /*T*/, const double* tau_host_unique, int n_u,
                        const int32_t* mod_id, double fps, bool grads, bool head, void* out);
    template <class T>
    void backward_sample(const void* dV);
    void check_comms();          // asynchronous NCCL errors -> NcclError
    void use_block_slot(int i);  // per-block recompute: point the shared activation slot at block i's kept O / lse
    template <class T>
    void block_fwd(int i, int64_t N);
    template <class T>
    void block_bwd(int i, int64_t N);
    template <class T>
    void block_fwd_tp(int i, int64_t N);
    template <class T>
    void block_bwd_tp(int i, int64_t N);
    std::vector<int> tp_ranks() const;  // the TP ranks this process computes
    void tp_allreduce(float* buf, int64_t n, cudaStream_t s);
    void tp_allreduce_grads(cudaStream_t s);
    template <class T>
    void sample_impl(const double* x_start, int64_t N, const int32_t* coords, const int64_t dims[3],
                     const double* text, int64_t L, const uint8_t* cond, const double* cond_latents, int64_t steps,
                     int direction, double fps, double* out);
    template <class T>
    void velocity_graph_impl(const double* rows, int64_t N, const int32_t* coords, const int64_t dims[3],
                             const double* text, int64_t L, const double* tau, double fps, double* V_out,
                             double* const* taps_out, const double* dV, double* const* grads_out);
    template <class T>
    void value_forward(const double* in, int64_t N, const int32_t* coords, const int64_t dims[3],
                       const double* text, int64_t L, const double* tau, double fps, double* out, bool velocity);

    const DevParam& P(const std::string& name) const;
    // TP rank slot k of a parameter (k indexes tp_ranks(); replicated params: the whole tensor)
    const float* Ps(const std::string& name, int k) const;
    const void* Ws(const std::string& name, int k) const;
    float* Gs(const std::string& name, int k) const;
    int tp_slots() const { return tp_ > 1 && tp_virtual_ ? tp_ : 1; }
    const void* W(const std::string& name) const;  // GEMM operand in the compute precision
    float* G(const std::string& name) const;
    std::string blk(int i, const char* s) const { return "dit.blk." + std::to_string(i) + "." + s; }

    void plan_workspace(int64_t N, int64_t L, int n_u);

    int device_;
    bool bf16_;
    cudaStream_t stream_ = nullptr;
    Cfg cfg_;
    bool have_params_ = false;
    bool varlen_ = false;
    bool recompute_ = false;
    std::map<std::string, DevParam> params_;
    std::vector<DevParam*> sorted_;
    float* grad_buf_ = nullptr;
    int64_t grad_numel_ = 0;
    int64_t repl_numel_ = 0;  // TP: the replicated parameters' leading range of the gradient buffer
    const float* full_view(const DevParam& q, const float* local, float* a, float* b);
    Arena arena_;
    double last_ms_ = 0.0;
    int64_t last_launches_ = 0;
    Prof prof_;
    // NCCL data parallel.  The gradient all-reduce is bucketed: during the last local sample's backward the
    // FFN and cross-attention gradients of each block are all-reduced on dp_stream_ as soon as they are final
    // (overlapping the attention backward); dp_finish reduces the rest.  All DP collectives use dp_stream_.
    ncclComm_t comm_ = nullptr;
    int rank_ = 0, world_ = 1;
    cudaStream_t dp_stream_ = nullptr;
    bool dp_overlap_ = false;
    std::vector<std::pair<int64_t, int64_t>> dp_done_;  // (offset, length) of the buckets already reduced
    void dp_bucket(int block, const char* group);
    void dp_finish(double* scal);
    // AdamW state: m, v in the gradient buffer's layout; per-parameter table for the multi-tensor update
    struct Adam {
        bool on = false;
        double lr = 0, b1 = 0.9, b2 = 0.999, eps = 1e-8, wd = 0;
        int64_t step = 0;
    } adam_;
    float* opt_m_ = nullptr;
    float* opt_v_ = nullptr;
    void* param_table_ = nullptr;
    void alloc_adam_state();
    // tensor parallel
    ncclComm_t tp_comm_ = nullptr;
    int tp_ = 1, tp_rank_ = 0;
    bool tp_virtual_ = false;
    // peer-memory TP exchange (tp_peer.h); MGV_TP_EXCHANGE=nccl selects the NCCL all-reduce instead
    bool tp_peer_ = true;
    bool tpx_bf16_ = false;   // bf16 exchange payload (bf16 mode, MGV_TP_PAYLOAD=bf16)
    char* tpx_base_[8] = {};  // every rank's arena as mapped here (emulated ranks: slices of tpx_own_)
    char* tpx_own_ = nullptr;
    int64_t tpx_bytes_ = 0;   // capacity per rank arena
    uint64_t tpx_epoch_ = 0;
    bool tp_peer_on() const { return tp_ > 1 && tp_peer_; }
    void tp_peer_ensure(int64_t N);
    void tp_peer_release();
    float* tp_exchange(float* part, int64_t N, cudaStream_t s);

    // ---- per-sample workspace views (set by plan_workspace / forward)
public:
    struct WS;

private:
    WS* ws_ = nullptr;
};

}  // namespace mgv
