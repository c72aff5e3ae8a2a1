// DiT hot-path runtime: forward + backward of velocity_rows_graph and the flow
// loss for one sample at a time (samples are independent, dit.hpp:97-100), with
// gradient accumulation over the batch and an NCCL all-reduce for data
// parallelism.  Equations restate proj/src/dit.cpp:267-334;
// each step below cites the reference line it implements.
#include "model.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <unordered_map>

#include "attn.h"
#include "gemm.cuh"
#include "kernels.h"
#include "tp_peer.h"

namespace mgv {

#define MGV_NCCL(x)                                                                        \
    do {                                                                                   \
        ncclResult_t r_ = (x);                                                             \
        if (r_ != ncclSuccess) throw NcclError(std::string(#x) + ": " + ncclGetErrorString(r_)); \
    } while (0)

void validate_cfg(const Cfg& c) {  // dit.cpp:50-63
    if (c.depth < 1 || c.hidden < 1 || c.heads < 1 || c.text_dim < 1 || c.c_z < 1)
        throw ConfigError("dit config dims must be positive");
    if (c.hidden % c.heads != 0) throw ConfigError("hidden must be a multiple of heads");
    int64_t sum = 0;
    for (int d : c.rope) {
        if (d <= 0 || d % 2 != 0) throw ConfigError("rope_split parts must be positive and even");
        sum += d;
    }
    if (sum != c.hd()) throw ConfigError("rope_split must sum to head_dim " + std::to_string(c.hd()));
    if (c.hidden > 4096) throw ConfigError("hidden > 4096 is not supported by the row kernels");
    if (c.hd() > 192) throw ConfigError("head_dim > 192 is not supported");
}

// ------------------------------------------------------------------ arena
Arena::~Arena() {
    if (base_) cudaFree(base_);
}
void Arena::reserve(size_t bytes) {
    if (bytes <= cap_) return;
    if (base_) MGV_CUDA(cudaFree(base_));
    base_ = nullptr;
    cap_ = 0;
    MGV_CUDA(cudaMalloc(&base_, bytes));
    cap_ = bytes;
    off_ = 0;
}

// ------------------------------------------------------------------ workspace
struct Blk {
    float *X1, *X2, *r0, *r1, *r2, *rc, *iq, *ik, *lse, *lse_x;
    void *a, *qkv, *qk, *O, *ao, *cn, *cqs, *kv, *Ox, *co, *f, *z, *h, *ff;
    // transposed attention operands written by the producing GEMM epilogues (WS::tpose): rotated q | k, v, q'
    void *qkT = nullptr, *vT = nullptr, *cqT = nullptr;
};
struct Model::WS {
    int64_t N = 0, L = 0;
    int n_u = 0, esz = 4;
    bool grads = false;
    void* rows;
    float* vt;
    uint8_t* lmask;
    int32_t* mod_id;
    int32_t* coords;
    float2* cs;
    double *taus, *phi, *z_in, *h_in, *g;
    std::vector<double*> gb;
    std::vector<float*> table;
    void* text;
    std::vector<float*> X;
    std::vector<Blk> blk;
    float* rf;
    void *fin, *Y, *dV;
    float* V;
    // backward
    float* dX;
    void *sA, *sB, *s1, *s2, *dkv;
    float *Dvec, *part1, *part2, *dkv_part, *dm;
    double *dg, *dgb, *loss_part, *scal;
    int* cnt;
    int q_splits_x = 1;
    // tensor parallel: fp32 partial sums of the row-parallel GEMMs (the all-reduce buffer)
    int tp = 1, tp_slots = 1;  // slots: TP ranks whose per-rank activations live here (emulated ranks: all)
    float* tpp = nullptr;
    // varlen packing: per 128-row tile its sample's [start, end) (AttnProblem::seg); seg = null when unpacked
    int* segbuf = nullptr;
    const int* seg = nullptr;
    // bf16, unsharded: the attention operands' transposes ([heads*hd][ldT]) come from GEMM epilogues
    bool tpose = false;
    int64_t ldT = 0;
    // training with per-block activation recompute: one block's activations (slot 0), every block's input X kept,
    // and every block's self-attention output O and lse (the recompute re-runs the GEMMs and row kernels, not the
    // attention forward: O / lse are small next to what they cost to recompute)
    bool recompute = false;
    bool recompute_pass = false;  // set while re-running a block's forward inside the backward
    std::vector<void*> Okeep;
    std::vector<float*> lsekeep;
    void* dOT = nullptr;  // dO^T of the attention being differentiated (self, then cross)
};

struct AdamParam {
    float* w;
    __nv_bfloat16* wb;
    int64_t off, n;
};

namespace {
struct Sizer {  // measures then lays out the arena
    bool measure;
    size_t bytes = 0;
    Arena* arena;
    template <class T>
    T* take(int64_t n) {
        size_t b = (sizeof(T) * static_cast<size_t>(n) + 255) & ~size_t(255);
        bytes += b;
        return measure ? nullptr : arena->take<T>(n);
    }
    void* takeT(int64_t n, int esz) { return esz == 2 ? (void*)take<__nv_bfloat16>(n) : (void*)take<float>(n); }
};

template <class S>
void layout_ws(Model::WS& w, S& a, const Cfg& c, bool grads) {
    const int64_t N = w.N, L = w.L, H = c.H(), D = c.D(), nh = c.heads, hd = c.hd();
    const int64_t Hr = H / w.tp, R = w.tp > 1 ? w.tp_slots : 1;
    const int e = w.esz;
    const int nu = w.n_u;
    w.rows = a.takeT(N * D, e);
    w.vt = a.template take<float>(N * D);
    w.lmask = a.template take<uint8_t>(N);
    w.mod_id = a.template take<int32_t>(N);
    w.coords = a.template take<int32_t>(N * 3);
    w.cs = a.template take<float2>(N * hd / 2);
    w.taus = a.template take<double>(nu);
    w.phi = a.template take<double>((nu + 1) * 32);
    w.z_in = a.template take<double>((nu + 1) * H);
    w.h_in = a.template take<double>((nu + 1) * H);
    w.g = a.template take<double>((nu + 1) * H);
    w.gb.assign(c.depth, nullptr);
    w.table.assign(c.depth, nullptr);
    for (int i = 0; i < c.depth; ++i) {
        w.gb[i] = a.template take<double>(nu * H);
        w.table[i] = a.template take<float>(nu * 6 * H);
    }
    w.text = a.takeT(L * c.text_dim, e);
    const int nX = grads ? c.depth + 1 : 2;
    w.X.assign(nX, nullptr);
    for (int i = 0; i < nX; ++i) w.X[i] = a.template take<float>(N * H);
    const int nB = grads && !w.recompute ? c.depth : 1;
    w.blk.assign(nB, Blk{});
    for (int i = 0; i < nB; ++i) {
        Blk& b = w.blk[i];
        b.X1 = a.template take<float>(N * H);
        b.X2 = a.template take<float>(N * H);
        b.r0 = a.template take<float>(N);
        b.r1 = a.template take<float>(N);
        b.r2 = a.template take<float>(N);
        b.rc = a.template take<float>(N);
        b.iq = a.template take<float>(N * nh);
        b.ik = a.template take<float>(N * nh);
        b.lse = a.template take<float>(((N + 127) / 128 * 128) * nh);
        b.lse_x = a.template take<float>(((N + 127) / 128 * 128) * nh);
        // TP: the head / column-parallel activations are per rank (width H/P per slot, compact), the rest is
        // replicated; R slots are held here (a real rank: 1, emulated ranks: P)
        b.a = a.takeT(N * H, e);
        b.qkv = a.takeT(R * N * 3 * Hr, e);
        b.qk = a.takeT(R * N * 2 * Hr, e);
        b.O = a.takeT(R * N * Hr, e);
        b.ao = a.takeT(N * H, e);
        b.cn = a.takeT(N * H, e);
        b.cqs = a.takeT(R * N * Hr, e);
        b.kv = a.takeT(R * L * 2 * Hr, e);
        b.Ox = a.takeT(R * N * Hr, e);
        b.co = a.takeT(N * H, e);
        b.f = a.takeT(N * H, e);
        b.z = a.takeT(R * N * 4 * Hr, e);
        b.h = a.takeT(R * N * 4 * Hr, e);
        b.ff = a.takeT(N * H, e);
        if (w.tpose) {
            b.qkT = a.takeT(2 * H * w.ldT, 2);
            b.vT = a.takeT(H * w.ldT, 2);
            b.cqT = a.takeT(H * w.ldT, 2);
        }
    }
    w.Okeep.assign(grads && w.recompute ? c.depth : 0, nullptr);
    w.lsekeep.assign(grads && w.recompute ? c.depth : 0, nullptr);
    for (size_t i = 0; i < w.Okeep.size(); ++i) {
        w.Okeep[i] = a.takeT(R * N * Hr, e);
        w.lsekeep[i] = a.template take<float>(((N + 127) / 128 * 128) * nh);
    }
    w.segbuf = a.template take<int>(2 * ((N + 127) / 128));
    w.seg = nullptr;
    w.rf = a.template take<float>(N);
    w.fin = a.takeT(N * H, e);
    w.Y = a.takeT(N * H, e);
    w.V = a.template take<float>(N * D);
    w.dV = a.takeT(N * D, e);
    w.tpp = w.tp > 1 ? a.template take<float>(N * H) : nullptr;
    w.loss_part = a.template take<double>(row_chunks(N) + 1024);
    w.scal = a.template take<double>(8);
    w.cnt = a.template take<int>(8);
    if (grads) {
        const int chunks = row_chunks(N);
        w.dX = a.template take<float>(N * H);
        w.sA = a.takeT(R * N * 4 * Hr, e);
        w.sB = a.takeT(R * N * 3 * Hr, e);
        w.s1 = a.takeT(N * H, e);
        w.s2 = a.takeT(N * H, e);
        w.dkv = a.takeT(R * L * 2 * Hr, e);
        if (w.tpose) w.dOT = a.takeT(H * w.ldT, 2);
        w.Dvec = a.template take<float>(((N + 127) / 128 * 128) * nh);
        // column partials: up to 4H wide, or one H-wide row per modulation-table row (n_u, a packed batch: B + 1)
        w.part1 = a.template take<float>((int64_t)chunks * std::max<int64_t>(4 * H, (int64_t)nu * H));
        w.part2 = a.template take<float>((int64_t)chunks * std::max<int64_t>(4 * H, (int64_t)nu * H));
        w.q_splits_x = static_cast<int>(std::min<int64_t>(64, (N + 31) / 32));
        w.dkv_part = a.template take<float>((int64_t)w.q_splits_x * nh * L * 2 * hd);
        w.dm = a.template take<float>(nu * 6 * H);
        w.dg = a.template take<double>(nu * H);
        w.dgb = a.template take<double>(nu * H);
    }
}
}  // namespace

void Model::plan_workspace(int64_t N, int64_t L, int n_u) {
    // (called through the templated entry points with ws_ fields preset)
    (void)N;
    (void)L;
    (void)n_u;
}

// ------------------------------------------------------------------ profiler
cudaEvent_t Prof::get() {
    cudaEvent_t e;
    if (!pool_.empty()) {
        e = pool_.back();
        pool_.pop_back();
    } else {
        MGV_CUDA(cudaEventCreate(&e));
    }
    used_.push_back(e);
    return e;
}
// The bf16 GEMMs of a profiled step are timed as one "gemm" phase (nested inside blocks_fwd / blocks_bwd).
static Prof* g_gemm_prof = nullptr;
static void gemm_prof_hook(bool begin, double flops, cudaStream_t s) {
    if (!g_gemm_prof) return;
    if (begin)
        g_gemm_prof->begin("gemm", s, flops);
    else
        g_gemm_prof->end(s);
}
GemmProfGuard::GemmProfGuard(Prof& p) {
    if (p.on) {
        g_gemm_prof = &p;
        g_gemm_prof_hook = gemm_prof_hook;
    }
}
GemmProfGuard::~GemmProfGuard() {
    g_gemm_prof = nullptr;
    g_gemm_prof_hook = nullptr;
}

void Prof::begin(const char* name, cudaStream_t s, double work) {
    if (!on) return;
    Pend p{name, get(), nullptr, work};
    MGV_CUDA(cudaEventRecord(p.a, s));
    pend_.push_back(p);
}
void Prof::end(cudaStream_t s) {
    if (!on) return;
    for (auto it = pend_.rbegin(); it != pend_.rend(); ++it)
        if (!it->b) {
            it->b = get();
            MGV_CUDA(cudaEventRecord(it->b, s));
            return;
        }
}
void Prof::end_step() {
    for (auto& p : pend_) {
        if (!p.b) continue;
        float ms = 0.0f;
        MGV_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
        Stat& st = stats[p.name];
        st.ms += ms;
        st.n += 1;
        st.work += p.work;
    }
    pend_.clear();
    for (auto e : used_) pool_.push_back(e);
    used_.clear();
}
Prof::~Prof() {
    for (auto e : pool_) cudaEventDestroy(e);
    for (auto e : used_) cudaEventDestroy(e);
}

__global__ void set_taus_kernel(double* taus, double t) {
    taus[0] = t;
    taus[1] = 0.0;
}
static void set_taus(double* taus, double t, cudaStream_t s) {
    set_taus_kernel<<<1, 1, 0, s>>>(taus, t);
    note_launch();
}

// ------------------------------------------------------------------ model
Model::Model(int device, bool bf16) : device_(device), bf16_(bf16) {
    MGV_CUDA(cudaSetDevice(device));
    // keep stream-ordered scratch (attention operand transposes) cached across steps
    cudaMemPool_t pool;
    MGV_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    MGV_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    ws_ = new WS();
}

Model::~Model() {
    cudaSetDevice(device_);
    for (auto& kv : params_) {
        if (kv.second.f32) cudaFree(kv.second.f32);
        if (kv.second.bf) cudaFree(kv.second.bf);
    }
    if (grad_buf_) cudaFree(grad_buf_);
    if (comm_) ncclCommDestroy(comm_);
    if (dp_stream_) cudaStreamDestroy(dp_stream_);
    tp_peer_release();
    if (tp_comm_) ncclCommDestroy(tp_comm_);
    if (opt_m_) cudaFree(opt_m_);
    if (opt_v_) cudaFree(opt_v_);
    if (param_table_) cudaFree(param_table_);
    delete ws_;
}

void Model::set_dp(int rank, int world, const uint8_t id[128]) {
    if (world < 1 || rank < 0 || rank >= world) throw InputError("bad data-parallel rank/world");
    if (comm_) {
        ncclCommDestroy(comm_);
        comm_ = nullptr;
    }
    rank_ = rank;
    world_ = world;
    // no id: no communicator.  world 1 is the plain context; world > 1 makes this context ONE rank's share of a
    // data-parallel step (loss and gradients scaled by 1 / global batch, not reduced): the sum over the ranks
    // is the global step, for external reducers and the decomposition test.  world 1 with an id: a one-rank
    // communicator (exercises the NCCL path).
    if (!id) return;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    MGV_CUDA(cudaSetDevice(device_));
    MGV_NCCL(ncclCommInitRank(&comm_, world, uid, rank));
    if (!dp_stream_) {  // highest priority: the all-reduce CTAs are dispatched ahead of pending attention CTAs
        int least = 0, greatest = 0;
        MGV_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        MGV_CUDA(cudaStreamCreateWithPriority(&dp_stream_, cudaStreamNonBlocking, greatest));
    }
}

// Gradient buckets of the data-parallel all-reduce (see model.h).  Names are sorted, so one block's
// "dit.blk.<i>.<group>" parameters are one contiguous range of the gradient buffer.
// Failure detection for the multi-GPU paths: a peer that died or a network error leaves an asynchronous error on
// the communicator; surface it as NcclError at the end of the step (the ABI returns MGV_ERR_NCCL) instead of letting
// the next collective hang.
void Model::check_comms() {
    for (ncclComm_t c : {comm_, tp_comm_}) {
        if (!c) continue;
        ncclResult_t r = ncclSuccess;
        MGV_NCCL(ncclCommGetAsyncError(c, &r));
        if (r != ncclSuccess && r != ncclInProgress)
            throw NcclError(std::string("asynchronous NCCL error on a ") + (c == comm_ ? "data" : "tensor") +
                            "-parallel communicator: " + ncclGetErrorString(r));
    }
}

void Model::dp_bucket(int block, const char* group) {
    if (!dp_overlap_) return;
    const std::string pre = "dit.blk." + std::to_string(block) + "." + group;
    int64_t lo = -1, hi = -1;
    for (const DevParam* q : sorted_)
        if (q->name.compare(0, pre.size(), pre) == 0) {
            if (lo < 0) lo = q->grad_off;
            hi = q->grad_off + q->numel;
        }
    if (lo < 0) return;
    cudaEvent_t ev;
    MGV_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    MGV_CUDA(cudaEventRecord(ev, stream_));
    MGV_CUDA(cudaStreamWaitEvent(dp_stream_, ev, 0));
    MGV_CUDA(cudaEventDestroy(ev));
    MGV_NCCL(ncclAllReduce(grad_buf_ + lo, grad_buf_ + lo, hi - lo, ncclFloat, ncclSum, comm_, dp_stream_));
    dp_done_.emplace_back(lo, hi - lo);
}

// The rest of the gradient buffer (every range no bucket covered) and the loss, then the step stream
// waits for all DP collectives.
void Model::dp_finish(double* scal) {
    cudaEvent_t ev;
    MGV_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    MGV_CUDA(cudaEventRecord(ev, stream_));
    MGV_CUDA(cudaStreamWaitEvent(dp_stream_, ev, 0));
    std::vector<std::pair<int64_t, int64_t>> done = dp_done_;
    std::sort(done.begin(), done.end());
    MGV_NCCL(ncclGroupStart());
    int64_t at = 0;
    for (const auto& d : done) {
        if (d.first > at) MGV_NCCL(ncclAllReduce(grad_buf_ + at, grad_buf_ + at, d.first - at, ncclFloat, ncclSum, comm_, dp_stream_));
        at = std::max(at, d.first + d.second);
    }
    if (at < grad_numel_)
        MGV_NCCL(ncclAllReduce(grad_buf_ + at, grad_buf_ + at, grad_numel_ - at, ncclFloat, ncclSum, comm_, dp_stream_));
    MGV_NCCL(ncclAllReduce(scal, scal, 1, ncclDouble, ncclSum, comm_, dp_stream_));
    MGV_NCCL(ncclGroupEnd());
    MGV_CUDA(cudaEventRecord(ev, dp_stream_));
    MGV_CUDA(cudaStreamWaitEvent(stream_, ev, 0));
    MGV_CUDA(cudaEventDestroy(ev));
    dp_done_.clear();
}

void Model::set_tp(int size, int rank, const uint8_t* id) {
    if (size < 1 || rank < 0 || rank >= size) throw InputError("bad tensor-parallel rank/size");
    if (have_params_ && size != tp_) throw ConfigError("set_tp must precede the parameter upload");
    if (tp_comm_) {
        ncclCommDestroy(tp_comm_);
        tp_comm_ = nullptr;
    }
    tp_peer_release();
    tpx_epoch_ = 0;
    if (const char* x = std::getenv("MGV_TP_EXCHANGE")) tp_peer_ = std::strcmp(x, "nccl") != 0;
    const char* pay = std::getenv("MGV_TP_PAYLOAD");
    tpx_bf16_ = bf16_ && pay && std::strcmp(pay, "bf16") == 0;
    tp_ = size;
    tp_rank_ = id ? rank : 0;
    tp_virtual_ = id == nullptr;
    if (size == 1 || !id) return;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    MGV_CUDA(cudaSetDevice(device_));
    MGV_NCCL(ncclCommInitRank(&tp_comm_, size, uid, rank));
}

std::vector<int> Model::tp_ranks() const {
    std::vector<int> r;
    if (tp_virtual_)
        for (int v = 0; v < tp_; ++v) r.push_back(v);
    else
        r.push_back(tp_rank_);
    return r;
}

void Model::tp_allreduce(float* buf, int64_t n, cudaStream_t s) {
    if (tp_ == 1 || tp_virtual_) return;  // emulated ranks accumulate the partials in place
    prof_.begin("tp_allreduce", s);
    MGV_NCCL(ncclAllReduce(buf, buf, n, ncclFloat, ncclSum, tp_comm_, s));
    prof_.end(s);
}

// ---- peer-memory TP exchange (protocol in tp_peer.h)
static int64_t tpx_rpr(int64_t N, int P) { return (N + P - 1) / P; }
// esz: payload bytes per element (4 fp32, 2 bf16)
static char* tpx_mbox(char* base) { return base + kTpFlagBytes; }
static char* tpx_result(char* base, int P, int64_t rpr, int64_t H, int esz) { return tpx_mbox(base) + P * rpr * H * esz; }
static unsigned long long* tpx_flags(char* base, int phase) {
    return reinterpret_cast<unsigned long long*>(base) + phase * kMaxTp;
}

// epilogue of rank src's row-parallel GEMM: its rows of owner o go to slot src of o's mailbox
static EpiF32Peer tp_epi(char* const* base, int P, int src, float alpha, int64_t N, int64_t H, bool bf16) {
    const int64_t rpr = tpx_rpr(N, P);
    const int esz = bf16 ? 2 : 4;
    EpiF32Peer e{};
    for (int o = 0; o < P; ++o) e.box[o] = tpx_mbox(base[o]) + src * rpr * H * esz;
    e.bf16 = bf16 ? 1 : 0;
    e.ldo = H;
    e.alpha = alpha;
    e.rpr = static_cast<int>(rpr);
    e.M = static_cast<int>(N);
    e.N = static_cast<int>(H);
    return e;
}

void Model::tp_peer_release() {
    if (!tpx_own_) return;
    cudaSetDevice(device_);
    if (!tp_virtual_)
        for (int o = 0; o < tp_; ++o)
            if (o != tp_rank_ && tpx_base_[o]) cudaIpcCloseMemHandle(tpx_base_[o]);
    cudaFree(tpx_own_);
    tpx_own_ = nullptr;
    tpx_bytes_ = 0;
    for (char*& b : tpx_base_) b = nullptr;
}

// Collective over the TP group when the arena grows (every rank runs the same N).  The arena of each rank
// holds flags + mailbox + result for rpr = ceil(N/P) rows; real ranks map each other's arenas with CUDA IPC,
// the handles travel over the TP communicator.
void Model::tp_peer_ensure(int64_t N) {
    if (!tp_peer_on()) return;
    const int P = tp_;
    const int64_t H = cfg_.H();
    if (H % (tpx_bf16_ ? 8 : 4) != 0) throw ConfigError("the peer-memory TP exchange needs hidden % 4 == 0 (bf16 payload: % 8)");
    const int64_t need = kTpFlagBytes + 2 * P * tpx_rpr(N, P) * H * (tpx_bf16_ ? 2 : 4);
    if (need <= tpx_bytes_) return;
    MGV_CUDA(cudaSetDevice(device_));
    MGV_CUDA(cudaStreamSynchronize(stream_));
    if (tpx_own_ && !tp_virtual_) {  // peers must be done with the old arenas before they go away
        float* one = nullptr;
        MGV_CUDA(cudaMalloc(&one, sizeof(float)));
        MGV_NCCL(ncclAllReduce(one, one, 1, ncclFloat, ncclSum, tp_comm_, stream_));
        MGV_CUDA(cudaStreamSynchronize(stream_));
        cudaFree(one);
    }
    tp_peer_release();
    const int copies = tp_virtual_ ? P : 1;
    MGV_CUDA(cudaMalloc(&tpx_own_, need * copies));
    MGV_CUDA(cudaMemset(tpx_own_, 0, need * copies));
    MGV_CUDA(cudaDeviceSynchronize());
    tpx_bytes_ = need;
    tpx_epoch_ = 0;
    if (tp_virtual_) {
        for (int o = 0; o < P; ++o) tpx_base_[o] = tpx_own_ + o * need;
        return;
    }
    cudaIpcMemHandle_t mine;
    MGV_CUDA(cudaIpcGetMemHandle(&mine, tpx_own_));
    const size_t hb = sizeof(cudaIpcMemHandle_t);
    char* dev = nullptr;
    MGV_CUDA(cudaMalloc(&dev, hb * P));
    MGV_CUDA(cudaMemcpy(dev + hb * tp_rank_, &mine, hb, cudaMemcpyHostToDevice));
    MGV_NCCL(ncclAllGather(dev + hb * tp_rank_, dev, hb, ncclChar, tp_comm_, stream_));
    std::vector<cudaIpcMemHandle_t> all(P);
    MGV_CUDA(cudaStreamSynchronize(stream_));
    MGV_CUDA(cudaMemcpy(all.data(), dev, hb * P, cudaMemcpyDeviceToHost));
    cudaFree(dev);
    for (int o = 0; o < P; ++o) {
        if (o == tp_rank_) {
            tpx_base_[o] = tpx_own_;
            continue;
        }
        void* p = nullptr;
        MGV_CUDA(cudaIpcOpenMemHandle(&p, all[o], cudaIpcMemLazyEnablePeerAccess));
        tpx_base_[o] = static_cast<char*>(p);
    }
}

// The exchange after the row-parallel GEMMs (whose epilogues already wrote the mailboxes): returns the
// summed N x H fp32 partial (peer mode: this rank's result region; NCCL mode: `part`, all-reduced in place).
float* Model::tp_exchange(float* part, int64_t N, cudaStream_t s) {
    if (!tp_peer_on()) {
        tp_allreduce(part, N * cfg_.H(), s);
        return part;
    }
    prof_.begin("tp_exchange", s);
    const int P = tp_;
    const int64_t H = cfg_.H(), rpr = tpx_rpr(N, P);
    const int esz = tpx_bf16_ ? 2 : 4;
    const uint64_t e = ++tpx_epoch_;
    const std::vector<int> ranks = tp_ranks();
    auto signal = [&](int src, int phase) {
        TpFlagPtrs f{};
        for (int o = 0; o < P; ++o) f.f[o] = tpx_flags(tpx_base_[o], phase) + src;
        tp_signal(f, P, e, s);
    };
    for (int k : ranks) signal(k, 0);
    for (int k : ranks) {
        const int64_t rows = std::max<int64_t>(0, std::min<int64_t>(rpr, N - k * rpr));
        TpDstPtrs d{};
        int nd = 0;
        if (tp_virtual_)  // emulated ranks share one set of activation buffers: one result region
            d.p[nd++] = tpx_result(tpx_base_[0], P, rpr, H, esz) + k * rpr * H * esz;
        else
            for (int j = 0; j < P; ++j) d.p[nd++] = tpx_result(tpx_base_[j], P, rpr, H, esz) + k * rpr * H * esz;
        tp_reduce_gather(tpx_mbox(tpx_base_[k]), tpx_bf16_, P, rpr, rows, H, d, nd, tpx_flags(tpx_base_[k], 0), e, s);
    }
    for (int k : ranks) signal(k, 1);
    for (int k : ranks) tp_wait(tpx_flags(tpx_base_[k], 1), P, e, s);
    char* res = tpx_result(tpx_base_[tp_virtual_ ? 0 : tp_rank_], P, rpr, H, esz);
    if (tpx_bf16_) {  // the block's consumers read the fp32 sum: widen this rank's copy in place of `part`
        tp_bf16_to_f32(res, N * H, part, s);
        prof_.end(s);
        return part;
    }
    prof_.end(s);
    return reinterpret_cast<float*>(res);
}

// Shard map (expansion.cpp:143-180 chunk layout): row-parallel parameters are stored rank-major
// (rank r's rows of every chunk contiguous), column-parallel weights as P compact (rows x cols/P) blocks; a real
// TP rank holds only its own block, emulated ranks hold all P.  The rest is replicated.  Every rank computes its
// blocks' gradients alone, and the replicated gradients identically from the exchanged activations, so no
// gradient all-reduce is needed under TP.
static int tp_shard_kind(const std::string& n) {
    if (n.rfind("dit.blk.", 0) != 0) return 0;
    auto ends = [&](const char* m) {
        const size_t l = std::strlen(m);
        return n.size() >= l && n.compare(n.size() - l, l, m) == 0;
    };
    if (ends(".attn.out.w") || ends(".xattn.out.w") || ends(".ffn.out.w")) return 2;
    static const char* rows[] = {".attn.qkv.w", ".attn.qkv.b", ".attn.temp", ".xattn.q.w", ".xattn.q.b",
                                 ".xattn.kv.w", ".xattn.kv.b", ".ffn.in.w", ".ffn.in.b"};
    for (const char* m : rows)
        if (ends(m)) return 1;
    return 0;
}
void Model::tp_allreduce_grads(cudaStream_t) {}  // sharded storage: nothing to reduce (see tp_shard_kind)

// Chunked row layouts re-ordered rank-major under TP, so each rank's rows of every chunk are
// contiguous (qkv: chunks q|k|v, expansion.cpp:143-180 chunk layout; xattn.kv: k|v).
static int tp_row_chunks(const std::string& n) {
    auto ends = [&](const char* m) {
        const size_t l = std::strlen(m);
        return n.size() >= l && n.compare(n.size() - l, l, m) == 0;
    };
    if (n.rfind("dit.blk.", 0) != 0) return 0;
    if (ends(".attn.qkv.w") || ends(".attn.qkv.b")) return 3;
    if (ends(".xattn.kv.w") || ends(".xattn.kv.b")) return 2;
    return 0;
}

void Model::set_adamw(double lr, double beta1, double beta2, double eps, double weight_decay) {
    if (!(beta1 >= 0.0 && beta1 < 1.0 && beta2 >= 0.0 && beta2 < 1.0 && eps >= 0.0 && weight_decay >= 0.0))
        throw ConfigError("AdamW hyper-parameters out of range");
    adam_.on = lr > 0.0;
    adam_.lr = lr;
    adam_.b1 = beta1;
    adam_.b2 = beta2;
    adam_.eps = eps;
    adam_.wd = weight_decay;
    adam_.step = 0;
    if (adam_.on && have_params_) alloc_adam_state();
}

void Model::alloc_adam_state() {
    MGV_CUDA(cudaSetDevice(device_));
    if (!opt_m_) MGV_CUDA(cudaMalloc(&opt_m_, sizeof(float) * grad_numel_));
    if (!opt_v_) MGV_CUDA(cudaMalloc(&opt_v_, sizeof(float) * grad_numel_));
    MGV_CUDA(cudaMemsetAsync(opt_m_, 0, sizeof(float) * grad_numel_, stream_));
    MGV_CUDA(cudaMemsetAsync(opt_v_, 0, sizeof(float) * grad_numel_, stream_));
    MGV_CUDA(cudaStreamSynchronize(stream_));
}

// Multi-tensor AdamW (optim.cpp:7-24), one grid row per parameter: m, v, w updated in place, the bf16
// operand copy refreshed.  Skipped entirely when the step's loss is not finite (FlowTrainer::step throws
// before AdamW::update, flowtrain.cpp:276).
__device__ __forceinline__ float adamw_one(float gi, float& mi, float& vi, float wi, float lr, float b1, float b2,
                                           float eps, float wd, float inv_bc1, float inv_bc2) {
    mi = b1 * mi + (1.0f - b1) * gi;
    vi = b2 * vi + (1.0f - b2) * gi * gi;
    const float mh = mi * inv_bc1, vh = vi * inv_bc2;
    return wi - lr * (mh / (sqrtf(vh) + eps) + wd * wi);
}

// 16-byte accesses (the gradient / moment slices start at multiples of 64 elements, weights are cudaMalloc'd);
// per-element arithmetic is the scalar formula, so results do not depend on the vector width.
__global__ void adamw_kernel(const AdamParam* table, const float* grad, float* m, float* v, const double* loss_acc,
                             float lr, float b1, float b2, float eps, float wd, float inv_bc1, float inv_bc2) {
    if (!isfinite(*loss_acc)) return;
    const AdamParam q = table[blockIdx.y];
    const float4* g4 = reinterpret_cast<const float4*>(grad + q.off);
    float4* m4 = reinterpret_cast<float4*>(m + q.off);
    float4* v4 = reinterpret_cast<float4*>(v + q.off);
    float4* w4 = reinterpret_cast<float4*>(q.w);
    const int64_t n4 = q.n / 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n4; e += stride) {
        const float4 g = g4[e];
        float4 mm = m4[e], vv = v4[e], w = w4[e];
        w.x = adamw_one(g.x, mm.x, vv.x, w.x, lr, b1, b2, eps, wd, inv_bc1, inv_bc2);
        w.y = adamw_one(g.y, mm.y, vv.y, w.y, lr, b1, b2, eps, wd, inv_bc1, inv_bc2);
        w.z = adamw_one(g.z, mm.z, vv.z, w.z, lr, b1, b2, eps, wd, inv_bc1, inv_bc2);
        w.w = adamw_one(g.w, mm.w, vv.w, w.w, lr, b1, b2, eps, wd, inv_bc1, inv_bc2);
        m4[e] = mm;
        v4[e] = vv;
        w4[e] = w;
        if (q.wb) {
            __nv_bfloat162* b2p = reinterpret_cast<__nv_bfloat162*>(q.wb + 4 * e);
            b2p[0] = __floats2bfloat162_rn(w.x, w.y);
            b2p[1] = __floats2bfloat162_rn(w.z, w.w);
        }
    }
    for (int64_t e = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < q.n; e += stride) {  // tail
        float mi = m[q.off + e], vi = v[q.off + e];
        const float w = adamw_one(grad[q.off + e], mi, vi, q.w[e], lr, b1, b2, eps, wd, inv_bc1, inv_bc2);
        m[q.off + e] = mi;
        v[q.off + e] = vi;
        q.w[e] = w;
        if (q.wb) q.wb[e] = __float2bfloat16_rn(w);
    }
}

static bool is_matrix(const std::string& n) {
    static const char* mats[] = {"patch.w", "attn.qkv.w", "attn.out.w", "xattn.q.w", "xattn.kv.w",
                                 "xattn.out.w", "ffn.in.w", "ffn.out.w", "final.w", "out.w"};
    for (const char* m : mats) {
        const size_t l = std::strlen(m);
        if (n.size() >= l && n.compare(n.size() - l, l, m) == 0 && n.find("gmlp") == std::string::npos) return true;
    }
    return false;
}

__global__ void f64_to_f32_bf16(const double* src, int64_t n, float* f, __nv_bfloat16* b) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const float v = static_cast<float>(src[e]);
        f[e] = v;
        if (b) b[e] = __float2bfloat16_rn(v);
    }
}
__global__ void f32_to_f64(const float* src, int64_t n, double* dst) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        dst[e] = static_cast<double>(src[e]);
}
static int grid_of(int64_t n) { return static_cast<int>(std::min<int64_t>((n + 255) / 256, 1 << 20)); }

void Model::download_param(int64_t i, double* out) {
    if (i < 0 || i >= static_cast<int64_t>(sorted_.size())) throw InputError("parameter index out of range");
    MGV_CUDA(cudaSetDevice(device_));
    const DevParam& q = *sorted_[i];
    float *a = nullptr, *b = nullptr;
    double* d = nullptr;
    MGV_CUDA(cudaMallocAsync(&a, sizeof(float) * q.numel_full, stream_));
    MGV_CUDA(cudaMallocAsync(&b, sizeof(float) * q.numel_full, stream_));
    MGV_CUDA(cudaMallocAsync(&d, sizeof(double) * q.numel_full, stream_));
    const float* src = full_view(q, q.f32, a, b);
    f32_to_f64<<<grid_of(q.numel_full), 256, 0, stream_>>>(src, q.numel_full, d);
    note_launch();
    MGV_CUDA(cudaMemcpyAsync(out, d, sizeof(double) * q.numel_full, cudaMemcpyDeviceToHost, stream_));
    MGV_CUDA(cudaFreeAsync(a, stream_));
    MGV_CUDA(cudaFreeAsync(b, stream_));
    MGV_CUDA(cudaFreeAsync(d, stream_));
    MGV_CUDA(cudaStreamSynchronize(stream_));
}


void Model::upload(const Cfg& cfg, int64_t n, const char* const* names, const void* const* data,
                   const uint8_t* is_f32, const int64_t* numel) {
    validate_cfg(cfg);
    if (bf16_ && (cfg.hd() % 16 != 0 || cfg.text_dim % 8 != 0 || cfg.D() % 8 != 0))  // TMA rows / UMMA shapes
        throw ConfigError("bf16 tensor-core mode needs head_dim % 16 == 0 and text_dim, 4 c_z multiples of 8 "
                          "(use the fp32 parity mode for other shapes)");
    if (tp_ > 1 && (cfg.heads % tp_ != 0 || (cfg.hidden / tp_) % 8 != 0))
        throw ConfigError("tensor parallel size must divide heads, with hidden/size a multiple of 8");
    MGV_CUDA(cudaSetDevice(device_));
    const int64_t H = cfg.hidden, D = cfg.D();
    // expected dit.* names and shapes (dit.cpp:143-183)
    std::map<std::string, std::vector<int64_t>> want;
    want["dit.patch.w"] = {H, D};
    want["dit.patch.b"] = {H};
    want["dit.gmlp.in.w"] = {H, 32};
    want["dit.gmlp.in.b"] = {H};
    want["dit.gmlp.out.w"] = {H, H};
    want["dit.gmlp.out.b"] = {H};
    want["dit.mod.w"] = {6 * H, H};
    want["dit.mod.b"] = {6 * H};
    for (int i = 0; i < cfg.depth; ++i) {
        auto b = [&](const char* s) { return "dit.blk." + std::to_string(i) + "." + s; };
        want[b("gscale")] = {H};
        want[b("attn.qkv.w")] = {3 * H, H};
        want[b("attn.qkv.b")] = {3 * H};
        want[b("attn.temp")] = {cfg.heads};
        want[b("attn.out.w")] = {H, H};
        want[b("attn.out.b")] = {H};
        want[b("xattn.prenorm.g")] = {H};
        want[b("xattn.q.w")] = {H, H};
        want[b("xattn.q.b")] = {H};
        want[b("xattn.kv.w")] = {2 * H, cfg.text_dim};
        want[b("xattn.kv.b")] = {2 * H};
        want[b("xattn.out.w")] = {H, H};
        want[b("xattn.out.b")] = {H};
        want[b("xattn.postnorm.g")] = {H};
        want[b("ffn.in.w")] = {4 * H, H};
        want[b("ffn.in.b")] = {4 * H};
        want[b("ffn.out.w")] = {H, 4 * H};
        want[b("ffn.out.b")] = {H};
    }
    want["dit.final.g"] = {H};
    want["dit.final.w"] = {H, H};
    want["dit.final.b"] = {H};
    want["dit.out.w"] = {D, H};
    want["dit.out.b"] = {D};
    std::map<std::string, int64_t> given;
    for (int64_t i = 0; i < n; ++i) {
        std::string nm(names[i]);
        if (nm.rfind("dit.", 0) != 0) continue;  // register_params(..., "dit.") (flowtrain.cpp:260)
        given[nm] = i;
    }
    for (auto& kv : want)
        if (!given.count(kv.first)) throw InputError("no parameter named \"" + kv.first + "\"");  // params.cpp:24-28
    // (re)allocate when the configuration changed
    const bool same = have_params_ && cfg.depth == cfg_.depth && cfg.hidden == cfg_.hidden &&
                      cfg.heads == cfg_.heads && cfg.text_dim == cfg_.text_dim && cfg.c_z == cfg_.c_z;
    if (!same) {
        for (auto& kv : params_) {
            if (kv.second.f32) cudaFree(kv.second.f32);
            if (kv.second.bf) cudaFree(kv.second.bf);
        }
        params_.clear();
        sorted_.clear();
        if (grad_buf_) cudaFree(grad_buf_);
        grad_buf_ = nullptr;
        for (auto& kv : want) {
            DevParam p;
            p.name = kv.first;
            p.shape = kv.second;
            p.numel_full = 1;
            for (auto d : p.shape) p.numel_full *= d;
            p.shard = tp_ > 1 ? tp_shard_kind(p.name) : 0;
            p.slot_numel = p.shard ? p.numel_full / tp_ : p.numel_full;
            p.numel = p.shard && !tp_virtual_ ? p.slot_numel : p.numel_full;  // a real TP rank: its block only
            MGV_CUDA(cudaMalloc(&p.f32, sizeof(float) * p.numel));
            if (bf16_ && is_matrix(p.name)) MGV_CUDA(cudaMalloc(&p.bf, sizeof(__nv_bfloat16) * p.numel));
            params_[p.name] = p;
        }
        // gradient buffer: sorted names; under TP the replicated parameters first, then the sharded blocks (the
        // gradient norm sums the second range over the TP ranks)
        int64_t total = 0;
        for (int pass = 0; pass < 2; ++pass)
            for (auto& kv : params_) {
                if ((kv.second.shard != 0) != (pass == 1)) continue;
                kv.second.grad_off = total;
                total += (kv.second.numel + 63) / 64 * 64;
            }
        repl_numel_ = 0;
        for (auto& kv : params_)
            if (!kv.second.shard) repl_numel_ = std::max(repl_numel_, kv.second.grad_off + (kv.second.numel + 63) / 64 * 64);
        grad_numel_ = total;
        MGV_CUDA(cudaMalloc(&grad_buf_, sizeof(float) * total));
        for (auto& kv : params_) {
            kv.second.grad = grad_buf_ + kv.second.grad_off;
            sorted_.push_back(&kv.second);
        }
        std::vector<AdamParam> table;
        for (DevParam* q : sorted_) table.push_back(AdamParam{q->f32, q->bf, q->grad_off, q->numel});
        if (param_table_) cudaFree(param_table_);
        MGV_CUDA(cudaMalloc(&param_table_, sizeof(AdamParam) * table.size()));
        MGV_CUDA(cudaMemcpy(param_table_, table.data(), sizeof(AdamParam) * table.size(), cudaMemcpyHostToDevice));
        if (opt_m_) cudaFree(opt_m_);
        if (opt_v_) cudaFree(opt_v_);
        opt_m_ = opt_v_ = nullptr;
    }
    adam_.step = 0;  // new weights: fresh optimizer state (FlowTrainer owns a fresh AdamW)
    if (adam_.on) alloc_adam_state();
    cfg_ = cfg;
    double* staging = nullptr;
    int64_t stage_n = 0;
    for (auto& kv : params_) stage_n = std::max(stage_n, kv.second.numel_full);
    // staging: [0, n) fp64 input | [n, 2n) permuted rows (TP) | [2n, 3n) raw fp32 input (widened exactly)
    MGV_CUDA(cudaMalloc(&staging, sizeof(double) * stage_n * 3));
    for (auto& kv : params_) {
        DevParam& p = kv.second;
        const int64_t gi = given[p.name];
        const int64_t nf = p.numel_full;
        if (numel[gi] != nf)
            throw DimensionError("parameter " + p.name + " has " + std::to_string(numel[gi]) + " elements, expected " +
                                 std::to_string(nf));
        if (is_f32 && is_f32[gi]) {
            float* raw = reinterpret_cast<float*>(staging + 2 * stage_n);
            MGV_CUDA(cudaMemcpyAsync(raw, data[gi], sizeof(float) * nf, cudaMemcpyHostToDevice, stream_));
            f32_to_f64<<<grid_of(nf), 256, 0, stream_>>>(raw, nf, staging);
            ::mgv::note_launch();
        } else {
            MGV_CUDA(cudaMemcpyAsync(staging, data[gi], sizeof(double) * nf, cudaMemcpyHostToDevice, stream_));
        }
        const double* src = staging;  // to the rank-major shard layout
        if (const int C = p.shard == 1 ? tp_row_chunks(p.name) : 0) {
            permute_shard_rows(staging, staging + stage_n, C, static_cast<int>(H), tp_, nf / (C * H), 0, stream_);
            src = staging + stage_n;
        } else if (p.shard == 2) {
            permute_shard_cols(staging, staging + stage_n, p.shape[0], p.shape[1], tp_, 0, stream_);
            src = staging + stage_n;
        }
        if (p.shard && !tp_virtual_) src += tp_rank_ * p.slot_numel;  // this rank's block
        f64_to_f32_bf16<<<grid_of(p.numel), 256, 0, stream_>>>(src, p.numel, p.f32, p.bf); ::mgv::note_launch();
        MGV_CUDA(cudaGetLastError());
    }
    MGV_CUDA(cudaStreamSynchronize(stream_));
    cudaFree(staging);
    have_params_ = true;
}

const DevParam& Model::P(const std::string& name) const {
    auto it = params_.find(name);
    if (it == params_.end()) throw InputError("no parameter named \"" + name + "\"");
    return it->second;
}
const void* Model::W(const std::string& name) const {
    const DevParam& p = P(name);
    return bf16_ ? static_cast<const void*>(p.bf) : static_cast<const void*>(p.f32);
}
float* Model::G(const std::string& name) const { return P(name).grad; }
const float* Model::Ps(const std::string& name, int k) const {
    const DevParam& p = P(name);
    return p.f32 + (p.shard ? k * p.slot_numel : 0);
}
const void* Model::Ws(const std::string& name, int k) const {
    const DevParam& p = P(name);
    const int64_t o = p.shard ? k * p.slot_numel : 0;
    return bf16_ ? static_cast<const void*>(p.bf + o) : static_cast<const void*>(p.f32 + o);
}
float* Model::Gs(const std::string& name, int k) const {
    const DevParam& p = P(name);
    return p.grad + (p.shard ? k * p.slot_numel : 0);
}

// A parameter (or its gradient, `local` = the grad slice) as the full reference tensor, fp32, on the device:
// a real TP rank all-gathers the ranks' blocks (a collective over the TP group), then the shard layout is undone.
const float* Model::full_view(const DevParam& q, const float* local, float* a, float* b) {
    const float* src = local;
    if (q.shard && !tp_virtual_) {
        MGV_NCCL(ncclAllGather(local, a, q.slot_numel, ncclFloat, tp_comm_, stream_));
        src = a;
    }
    if (const int C = q.shard == 1 ? tp_row_chunks(q.name) : 0) {
        permute_shard_rows(src, b, C, static_cast<int>(cfg_.hidden), tp_, q.numel_full / (C * cfg_.hidden), 1,
                           stream_);
        return b;
    }
    if (q.shard == 2) {
        permute_shard_cols(src, b, q.shape[0], q.shape[1], tp_, 1, stream_);
        return b;
    }
    return src;
}

// ------------------------------------------------------------------ helpers
namespace {
inline Mat KM(const void* p, int64_t ld) { return Mat{p, ld, Major::K}; }
inline Mat MN(const void* p, int64_t ld) { return Mat{p, ld, Major::MN}; }
template <class T>
inline T* tp(void* p) { return static_cast<T*>(p); }
template <class T>
inline const T* tp(const void* p) { return static_cast<const T*>(p); }
template <class T>
inline void* off(void* p, int64_t n) { return static_cast<T*>(p) + n; }
template <class T>
inline const void* off(const void* p, int64_t n) { return static_cast<const T*>(p) + n; }
}  // namespace

// QKV projection + QK-L2-norm x temperature + 3-D RoPE (dit.cpp:288-294).  bf16 mode: one tcgen05 GEMM with
// BN = head_dim whose epilogue writes the raw q|k|v, the inverse norms and the rotated q|k (EpiQKNormRope,
// bit-identical to the GEMM + qk_norm_rope_vec pair it replaces); fp32 parity mode and head dims without a
// whole-head tile: the GEMM and the row kernel.
// fusion switches (tests / A-B only): bit 0 the QKV epilogue, bit 1 post-norm residual + FFN modulated RMSNorm,
// bit 2 the attention operands' transposes written by the producing GEMM epilogues (needs bit 0)
constexpr int kFuseQKV = 1, kFuseNormMod = 2, kFuseT = 4;
int g_fusions = kFuseQKV | kFuseNormMod | kFuseT;
extern "C" void mgv_dev_set_fusions(int mask) { g_fusions = mask; }
// bf16, unsharded, a head_dim with the fused QKV tile: Q^T / K^T / V^T / q'^T / dO^T come from GEMM epilogues
static void set_tpose(Model::WS& w, const Cfg& c) {
    const int64_t hd = c.hd();
    w.tpose = w.esz == 2 && w.tp == 1 && (g_fusions & kFuseT) && (g_fusions & kFuseQKV) &&
              (hd == 64 || hd == 128 || hd == 144) && c.H() % 8 == 0;
    w.ldT = w.tpose ? (w.N + 7) / 8 * 8 : 0;
}
template <int HD>
static bool qkv_fused_launch(const void* a, int64_t H, const void* Wq, const float* bias, int n, int64_t Hl,
                             const QKLayout& L, const float* temp, const float2* cs, void* qkv, void* qk, float* iq,
                             float* ik, void* qkT, void* vT, int64_t ldT, cudaStream_t s) {
    using bf = __nv_bfloat16;
    EpiQKNormRope<HD> e{static_cast<bf*>(qkv), L.in_ld, bias, static_cast<bf*>(qk), L.out_ld, L.out_koff, Hl, temp,
                        cs, iq, ik, L.i_ld, n, static_cast<bf*>(qkT), ldT};
    // q | k rows of the weight with the whole-head tile; the v rows keep the 256-wide tile (a 144-wide tile
    // moves 39% more shared-memory bytes per FLOP: its V third would cost more than it saves)
    gemm_tc_bn<HD>(KM(a, H), KM(Wq, H), n, static_cast<int>(2 * Hl), static_cast<int>(H), e, s);
    if (vT)
        gemm(true, KM(a, H), KM(static_cast<const bf*>(Wq) + 2 * Hl * H, H), n, static_cast<int>(Hl),
             static_cast<int>(H),
             EpiStoreT{static_cast<bf*>(qkv) + 2 * Hl, L.in_ld, bias + 2 * Hl, 1.0f, n, static_cast<int>(Hl),
                       static_cast<bf*>(vT), ldT},
             s);
    else
        gemm(true, KM(a, H), KM(static_cast<const bf*>(Wq) + 2 * Hl * H, H), n, static_cast<int>(Hl),
             static_cast<int>(H),
             EpiStore<bf>{static_cast<bf*>(qkv) + 2 * Hl, L.in_ld, bias + 2 * Hl, 1.0f, n, static_cast<int>(Hl)}, s);
    return true;
}
template <class T>
static void qkv_norm_rope(bool bf16, const void* a, int64_t H, const void* Wq, const float* bias, int n, int64_t Hl,
                          int64_t heads, const QKLayout& L, const float* temp, const float2* cs, void* qkv, void* qk,
                          float* iq, float* ik, cudaStream_t s, void* qkT = nullptr, void* vT = nullptr,
                          int64_t ldT = 0) {
    const int64_t hd = Hl / heads;
    if constexpr (std::is_same<T, __nv_bfloat16>::value) {
        const bool lay = L.in_ld == 3 * Hl && L.in_koff == Hl && (H % 8) == 0 && (L.out_ld % 8) == 0 &&
                         (L.out_koff % 8) == 0;
        if (bf16 && (g_fusions & kFuseQKV) && lay) {
            if (hd == 144) { qkv_fused_launch<144>(a, H, Wq, bias, n, Hl, L, temp, cs, qkv, qk, iq, ik, qkT, vT, ldT, s); return; }
            if (hd == 128) { qkv_fused_launch<128>(a, H, Wq, bias, n, Hl, L, temp, cs, qkv, qk, iq, ik, qkT, vT, ldT, s); return; }
            if (hd == 64) { qkv_fused_launch<64>(a, H, Wq, bias, n, Hl, L, temp, cs, qkv, qk, iq, ik, qkT, vT, ldT, s); return; }
        }
    }
    if (qkT || vT) throw std::logic_error("transposed q|k|v outputs need the fused QKV path");
    gemm(bf16, KM(a, H), KM(Wq, H), n, static_cast<int>(3 * Hl), static_cast<int>(H),
         EpiStore<T>{tp<T>(qkv), 3 * Hl, bias, 1.0f, n, static_cast<int>(3 * Hl)}, s);
    qk_norm_rope<T>(tp<T>(qkv), L, n, static_cast<int>(Hl), static_cast<int>(heads), temp, cs, tp<T>(qk), iq, ik, s);
}

template <class T>
static void attention_fwd(bool bf16, const AttnProblem& p, cudaStream_t s) {
    if (bf16 && attn_tc_supported(p.hd, p.Nk))
        attn_fwd_tc(p, s);
    else
        attn_fwd_simt<T>(p, s);
}
template <class T>
static void attention_bwd(bool bf16, const AttnBwdProblem& p, cudaStream_t s) {
    if (bf16 && attn_tc_supported(p.f.hd, p.f.Nk))
        attn_bwd_tc(p, s);
    else
        attn_bwd_simt<T>(p, s);
}

void Model::use_block_slot(int i) {
    WS& w = *ws_;
    if (!w.recompute) return;
    w.blk[0].O = w.Okeep[static_cast<size_t>(i)];
    w.blk[0].lse = w.lsekeep[static_cast<size_t>(i)];
}

// ------------------------------------------------------------------ block forward (dit.cpp:279-313)
template <class T>
void Model::block_fwd(int i, int64_t N) {
    if (tp_ > 1) return block_fwd_tp<T>(i, N);
    WS& w = *ws_;
    const bool bf = bf16_;
    cudaStream_t s = stream_;
    const int64_t H = cfg_.H(), nh = cfg_.heads, hd = cfg_.hd(), L = w.L;
    Blk& b = w.blk[w.grads && !w.recompute ? i : 0];
    const float* Xin = w.X[w.grads ? i : (i % 2)];
    float* Xout = w.X[w.grads ? i + 1 : ((i + 1) % 2)];
    const float* tab = w.table[i];
    const int64_t tld = 6 * H;
    const int n = static_cast<int>(N);
    // self-attention: a = rms(x)(1+sc1)+sh1 (dit.cpp:287)
    rms_mod<T>(Xin, n, H, tab, tld, 0, H, w.mod_id, tp<T>(b.a), b.r0, s);
    qkv_norm_rope<T>(bf, b.a, H, W(blk(i, "attn.qkv.w")), P(blk(i, "attn.qkv.b")).f32, n, H, nh, qk_layout_full(H, nh),
                     P(blk(i, "attn.temp")).f32, w.cs, b.qkv, b.qk, b.iq, b.ik, s, b.qkT, b.vT, w.ldT);  // dit.cpp:288-294
    AttnProblem ap{b.qk, 2 * H, off<T>(b.qk, H), 2 * H, off<T>(b.qkv, 2 * H), 3 * H, b.O, H, b.lse,
                   n, n, int(nh), int(hd)};
    ap.vt = b.vT;  // null: the attention kernel transposes V itself
    ap.vt_ld = w.ldT;
    prof_.begin("attn_fwd", s);
    ap.lse_ld = (N + 127) / 128 * 128;
    ap.seg = w.seg;
    if (!w.recompute_pass) attention_fwd<T>(bf, ap, s);  // mha (autodiff.cpp:755-793); kept O / lse on recompute
    prof_.end(s);
    gemm(bf, KM(b.O, H), KM(W(blk(i, "attn.out.w")), H), n, H, H,
         EpiGateResid<T>{Xin, b.X1, H, tp<T>(b.ao), H, P(blk(i, "attn.out.b")).f32, tab + 2 * H, tld, w.mod_id, n,
                         int(H)},
         s);  // x += ao * gt1 (dit.cpp:295-297)
    // cross-attention (dit.cpp:300-305)
    rms_gain<T>(b.X1, n, H, P(blk(i, "xattn.prenorm.g")).f32, tp<T>(b.cn), b.r1, s);
    const float xscale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(hd)));
    if (b.cqT)
        gemm(bf, KM(b.cn, H), KM(W(blk(i, "xattn.q.w")), H), n, H, H,
             EpiStoreT{tp<__nv_bfloat16>(b.cqs), H, P(blk(i, "xattn.q.b")).f32, xscale, n, int(H),
                       tp<__nv_bfloat16>(b.cqT), w.ldT},
             s);
    else
        gemm(bf, KM(b.cn, H), KM(W(blk(i, "xattn.q.w")), H), n, H, H,
             EpiStore<T>{tp<T>(b.cqs), H, P(blk(i, "xattn.q.b")).f32, xscale, n, int(H)}, s);
    gemm(bf, KM(w.text, cfg_.text_dim), KM(W(blk(i, "xattn.kv.w")), cfg_.text_dim), int(L), 2 * H, cfg_.text_dim,
         EpiStore<T>{tp<T>(b.kv), 2 * H, P(blk(i, "xattn.kv.b")).f32, 1.0f, int(L), int(2 * H)}, s);
    AttnProblem xp{b.cqs, H, b.kv, 2 * H, off<T>(b.kv, H), 2 * H, b.Ox, H, b.lse_x, n, int(L), int(nh), int(hd)};
    prof_.begin("xattn_fwd", s);
    xp.lse_ld = (N + 127) / 128 * 128;
    attention_fwd<T>(bf, xp, s);
    prof_.end(s);
    gemm(bf, KM(b.Ox, H), KM(W(blk(i, "xattn.out.w")), H), n, H, H,
         EpiStore<T>{tp<T>(b.co), H, P(blk(i, "xattn.out.b")).f32, 1.0f, n, int(H)}, s);
    // post-norm residual (dit.cpp:305) + the feed-forward's modulated RMSNorm (dit.cpp:308) in one pass
    if (!(g_fusions & kFuseNormMod) ||
        !postnorm_resid_mod<T>(b.X1, tp<T>(b.co), n, H, P(blk(i, "xattn.postnorm.g")).f32, b.X2, b.rc, tab, tld,
                               3 * H, 4 * H, w.mod_id, tp<T>(b.f), b.r2, s)) {
        postnorm_resid<T>(b.X1, tp<T>(b.co), n, H, P(blk(i, "xattn.postnorm.g")).f32, b.X2, b.rc, s);
        rms_mod<T>(b.X2, n, H, tab, tld, 3 * H, 4 * H, w.mod_id, tp<T>(b.f), b.r2, s);
    }
    // feed-forward (dit.cpp:308-311)
    gemm(bf, KM(b.f, H), KM(W(blk(i, "ffn.in.w")), H), n, 4 * H, H,
         EpiBiasSilu<T>{tp<T>(b.z), tp<T>(b.h), 4 * H, P(blk(i, "ffn.in.b")).f32, n, int(4 * H)}, s);
    gemm(bf, KM(b.h, 4 * H), KM(W(blk(i, "ffn.out.w")), 4 * H), n, H, 4 * H,
         EpiGateResid<T>{b.X2, Xout, H, tp<T>(b.ff), H, P(blk(i, "ffn.out.b")).f32, tab + 5 * H, tld, w.mod_id, n,
                         int(H)},
         s);
}

// ------------------------------------------------------------------ block backward
template <class T>
void Model::block_bwd(int i, int64_t N) {
    if (tp_ > 1) return block_bwd_tp<T>(i, N);
    WS& w = *ws_;
    const bool bf = bf16_;
    cudaStream_t s = stream_;
    const int64_t H = cfg_.H(), nh = cfg_.heads, hd = cfg_.hd(), L = w.L;
    const int n = static_cast<int>(N), nu = w.n_u, chunks = row_chunks(n);
    Blk& b = w.blk[w.recompute ? 0 : i];
    const float* Xin = w.X[i];
    const float* tab = w.table[i];
    const int64_t tld = 6 * H;
    float* dX = w.dX;
    float* dm = w.dm;
    // dO = d(out-proj input) into w.s2 (and dO^T into w.dOT when the attention operands come transposed)
    auto store_dO = [&](const Mat& A, const Mat& B, int rows, int64_t K) {
        if (w.tpose)
            gemm(bf, A, B, rows, int(H), int(K),
                 EpiStoreT{tp<__nv_bfloat16>(w.s2), H, nullptr, 1.0f, rows, int(H), tp<__nv_bfloat16>(w.dOT), w.ldT}, s);
        else
            gemm(bf, A, B, rows, int(H), int(K), EpiStore<T>{tp<T>(w.s2), H, nullptr, 1.0f, rows, int(H)}, s);
    };
    // ---- FFN (dit.cpp:308-311)
    gate_bwd<T>(dX, tp<T>(b.ff), tab, tld, 5 * H, w.mod_id, nu, n, H, tp<T>(w.s1), w.part1, w.part2, s);
    reduce_chunks_grouped(w.part1, chunks, nu, H, dm + 5 * H, 6 * H, 1.0f, 0, s);  // d gt2
    reduce_chunks(w.part2, chunks, H, G(blk(i, "ffn.out.b")), 1.0f, 1, s);
    gemm(bf, MN(w.s1, H), MN(b.h, 4 * H), H, 4 * H, n, EpiF32{G(blk(i, "ffn.out.w")), 4 * H, nullptr, 1.0f, 1, int(H), int(4 * H)}, s);
    gemm(bf, KM(w.s1, H), MN(W(blk(i, "ffn.out.w")), 4 * H), n, 4 * H, H,
         EpiSiluBwd<T>{tp<T>(w.sA), tp<T>(b.z), 4 * H, n, int(4 * H)}, s);  // dz = (dff W2) silu'(z)
    colsum<T>(tp<T>(w.sA), 4 * H, n, 4 * H, w.part1, s);
    reduce_chunks(w.part1, chunks, 4 * H, G(blk(i, "ffn.in.b")), 1.0f, 1, s);
    gemm(bf, MN(w.sA, 4 * H), MN(b.f, H), 4 * H, H, n, EpiF32{G(blk(i, "ffn.in.w")), H, nullptr, 1.0f, 1, int(4 * H), int(H)}, s);
    gemm(bf, KM(w.sA, 4 * H), MN(W(blk(i, "ffn.in.w")), H), n, H, 4 * H,
         EpiStore<T>{tp<T>(w.s1), H, nullptr, 1.0f, n, int(H)}, s);  // df
    rms_mod_bwd<T>(tp<T>(w.s1), b.X2, b.r2, tab, tld, 3 * H, 4 * H, w.mod_id, nu, n, H, dX, w.part1, w.part2, s);
    reduce_chunks_grouped(w.part1, chunks, nu, H, dm + 3 * H, 6 * H, 1.0f, 0, s);  // d sh2
    reduce_chunks_grouped(w.part2, chunks, nu, H, dm + 4 * H, 6 * H, 1.0f, 0, s);  // d sc2
    dp_bucket(i, "ffn.");  // ffn.* gradients are final: all-reduce them under the attention backward
    // ---- cross-attention (dit.cpp:300-305)
    postnorm_bwd<T>(dX, tp<T>(b.co), b.rc, P(blk(i, "xattn.postnorm.g")).f32, n, H, tp<T>(w.s1), w.part1, s);
    reduce_chunks(w.part1, chunks, H, G(blk(i, "xattn.postnorm.g")), 1.0f, 1, s);
    colsum<T>(tp<T>(w.s1), H, n, H, w.part1, s);
    reduce_chunks(w.part1, chunks, H, G(blk(i, "xattn.out.b")), 1.0f, 1, s);
    gemm(bf, MN(w.s1, H), MN(b.Ox, H), H, H, n, EpiF32{G(blk(i, "xattn.out.w")), H, nullptr, 1.0f, 1, int(H), int(H)}, s);
    store_dO(KM(w.s1, H), MN(W(blk(i, "xattn.out.w")), H), n, H);
    AttnBwdProblem xb{AttnProblem{b.cqs, H, b.kv, 2 * H, off<T>(b.kv, H), 2 * H, b.Ox, H, b.lse_x, n, int(L), int(nh), int(hd)},
                      w.s2, H, w.Dvec, w.s1, H, w.dkv, 2 * H, off<T>(w.dkv, H), 2 * H, w.dkv_part, w.q_splits_x};
    if (w.tpose) {  // q'^T from the forward's xattn.q epilogue, dO^T from the dgrad epilogue above
        xb.qt = b.cqT;
        xb.qt_ld = w.ldT;
        xb.dot = w.dOT;
        xb.dot_ld = w.ldT;
    }
    prof_.begin("xattn_bwd", s);
    xb.f.lse_ld = (N + 127) / 128 * 128;
    attention_bwd<T>(bf, xb, s);
    prof_.end(s);
    const float xscale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(hd)));
    gemm(bf, MN(w.dkv, 2 * H), MN(w.text, cfg_.text_dim), 2 * H, cfg_.text_dim, int(L),
         EpiF32{G(blk(i, "xattn.kv.w")), cfg_.text_dim, nullptr, 1.0f, 1, int(2 * H), int(cfg_.text_dim)}, s);
    colsum<T>(tp<T>(w.dkv), 2 * H, int(L), 2 * H, w.part1, s);
    reduce_chunks(w.part1, row_chunks(int(L)), 2 * H, G(blk(i, "xattn.kv.b")), 1.0f, 1, s);
    colsum<T>(tp<T>(w.s1), H, n, H, w.part1, s);
    reduce_chunks(w.part1, chunks, H, G(blk(i, "xattn.q.b")), xscale, 1, s);
    gemm(bf, MN(w.s1, H), MN(b.cn, H), H, H, n, EpiF32{G(blk(i, "xattn.q.w")), H, nullptr, xscale, 1, int(H), int(H)}, s);
    gemm(bf, KM(w.s1, H), MN(W(blk(i, "xattn.q.w")), H), n, H, H, EpiStore<T>{tp<T>(w.s2), H, nullptr, xscale, n, int(H)}, s);
    rms_gain_bwd<T>(tp<T>(w.s2), b.X1, b.r1, P(blk(i, "xattn.prenorm.g")).f32, n, H, dX, 1, w.part1, s);
    reduce_chunks(w.part1, chunks, H, G(blk(i, "xattn.prenorm.g")), 1.0f, 1, s);
    dp_bucket(i, "xattn.");
    // ---- self-attention (dit.cpp:287-297)
    gate_bwd<T>(dX, tp<T>(b.ao), tab, tld, 2 * H, w.mod_id, nu, n, H, tp<T>(w.s1), w.part1, w.part2, s);
    reduce_chunks_grouped(w.part1, chunks, nu, H, dm + 2 * H, 6 * H, 1.0f, 0, s);  // d gt1
    reduce_chunks(w.part2, chunks, H, G(blk(i, "attn.out.b")), 1.0f, 1, s);
    gemm(bf, MN(w.s1, H), MN(b.O, H), H, H, n, EpiF32{G(blk(i, "attn.out.w")), H, nullptr, 1.0f, 1, int(H), int(H)}, s);
    store_dO(KM(w.s1, H), MN(W(blk(i, "attn.out.w")), H), n, H);
    AttnBwdProblem ab{AttnProblem{b.qk, 2 * H, off<T>(b.qk, H), 2 * H, off<T>(b.qkv, 2 * H), 3 * H, b.O, H, b.lse, n, n, int(nh), int(hd)},
                      w.s2, H, w.Dvec, w.sB, 3 * H, off<T>(w.sB, H), 3 * H, off<T>(w.sB, 2 * H), 3 * H, nullptr, 1};
    if (w.tpose) {  // Q^T / K^T / V^T from the forward's QKV epilogues, dO^T from the dgrad epilogue above
        ab.qt = b.qkT;
        ab.qt_ld = w.ldT;
        ab.kt = off<__nv_bfloat16>(b.qkT, H * w.ldT);
        ab.kt_ld = w.ldT;
        ab.f.vt = b.vT;
        ab.f.vt_ld = w.ldT;
        ab.dot = w.dOT;
        ab.dot_ld = w.ldT;
    }
    prof_.begin("attn_bwd", s);
    ab.f.lse_ld = (N + 127) / 128 * 128;
    ab.f.seg = w.seg;
    attention_bwd<T>(bf, ab, s);
    prof_.end(s);
    qk_norm_rope_bwd<T>(tp<T>(w.sB), tp<T>(b.qkv), qk_layout_full(H, nh), n, H, nh, P(blk(i, "attn.temp")).f32, w.cs, b.iq, b.ik, w.part1, s);
    reduce_chunks(w.part1, chunks, nh, G(blk(i, "attn.temp")), 1.0f, 1, s);
    colsum<T>(tp<T>(w.sB), 3 * H, n, 3 * H, w.part1, s);
    reduce_chunks(w.part1, chunks, 3 * H, G(blk(i, "attn.qkv.b")), 1.0f, 1, s);
    gemm(bf, MN(w.sB, 3 * H), MN(b.a, H), 3 * H, H, n, EpiF32{G(blk(i, "attn.qkv.w")), H, nullptr, 1.0f, 1, int(3 * H), int(H)}, s);
    gemm(bf, KM(w.sB, 3 * H), MN(W(blk(i, "attn.qkv.w")), H), n, H, 3 * H, EpiStore<T>{tp<T>(w.s1), H, nullptr, 1.0f, n, int(H)}, s);
    rms_mod_bwd<T>(tp<T>(w.s1), Xin, b.r0, tab, tld, 0, H, w.mod_id, nu, n, H, dX, w.part1, w.part2, s);
    reduce_chunks_grouped(w.part1, chunks, nu, H, dm, 6 * H, 1.0f, 0, s);      // d sh1
    reduce_chunks_grouped(w.part2, chunks, nu, H, dm + H, 6 * H, 1.0f, 0, s);  // d sc1
    // ---- shared modulation head (dit.cpp:280-283)
    modulation_bwd(dm, w.gb[i], P("dit.mod.w").f32, nu, H, G("dit.mod.w"), G("dit.mod.b"), w.dgb, s);
    gscale_bwd(w.dgb, w.g, P(blk(i, "gscale")).f32, nu, H, G(blk(i, "gscale")), w.dg, s);
}

// ------------------------------------------------------------------ memory accounting (per rank)
// What one TP rank (or a single-device context, tp = 1) allocates for a training step over N tokens: the
// parameters (fp32 masters + bf16 operand copies), the gradient buffer, the AdamW moments, the step workspace
// (every block's saved activations) and the peer-exchange arena.  The same layout code the runtime uses, run in
// measure mode, so a plan needs no device (the 56-block stack at P = 8).
void plan_rank_bytes(const Cfg& c, bool bf16, int tp, int64_t N, int64_t L, int n_u, int train, int64_t out[5]) {
    validate_cfg(c);
    if (tp < 1 || c.heads % tp != 0) throw ConfigError("tensor parallel size must divide heads");
    const int64_t H = c.H(), D = c.D();
    auto rnd = [](int64_t n) { return (n + 63) / 64 * 64; };
    int64_t pf = 0, pb = 0, pg = 0;
    auto add = [&](const std::string& name, int64_t numel, bool mat) {
        const int64_t local = tp > 1 && tp_shard_kind(name) ? numel / tp : numel;
        pf += 4 * local;
        if (bf16 && mat) pb += 2 * local;
        pg += 4 * rnd(local);
    };
    add("dit.patch.w", H * D, true), add("dit.patch.b", H, false), add("dit.gmlp.in.w", H * 32, false);
    add("dit.gmlp.in.b", H, false), add("dit.gmlp.out.w", H * H, false), add("dit.gmlp.out.b", H, false);
    add("dit.mod.w", 6 * H * H, false), add("dit.mod.b", 6 * H, false);
    for (int i = 0; i < c.depth; ++i) {
        const std::string b = "dit.blk." + std::to_string(i) + ".";
        add(b + "gscale", H, false), add(b + "attn.qkv.w", 3 * H * H, true), add(b + "attn.qkv.b", 3 * H, false);
        add(b + "attn.temp", c.heads, false), add(b + "attn.out.w", H * H, true), add(b + "attn.out.b", H, false);
        add(b + "xattn.prenorm.g", H, false), add(b + "xattn.q.w", H * H, true), add(b + "xattn.q.b", H, false);
        add(b + "xattn.kv.w", 2 * H * c.text_dim, true), add(b + "xattn.kv.b", 2 * H, false);
        add(b + "xattn.out.w", H * H, true), add(b + "xattn.out.b", H, false), add(b + "xattn.postnorm.g", H, false);
        add(b + "ffn.in.w", 4 * H * H, true), add(b + "ffn.in.b", 4 * H, false), add(b + "ffn.out.w", 4 * H * H, true);
        add(b + "ffn.out.b", H, false);
    }
    add("dit.final.g", H, false), add("dit.final.w", H * H, true), add("dit.final.b", H, false);
    add("dit.out.w", D * H, true), add("dit.out.b", D, false);
    Model::WS w;
    w.N = N;
    w.L = L;
    w.n_u = n_u;
    w.esz = bf16 ? 2 : 4;
    w.grads = train != 0;
    w.recompute = (train & 2) != 0;
    w.tp = tp;
    w.tp_slots = 1;
    set_tpose(w, c);
    Sizer sz{true, 0, nullptr};
    layout_ws(w, sz, c, train);
    out[0] = pf + pb;                              // parameters
    out[1] = train ? pg : 0;                       // gradients
    out[2] = train ? 2 * pg : 0;                   // AdamW m, v
    out[3] = static_cast<int64_t>(sz.bytes);       // workspace (saved activations + scratch)
    out[4] = tp > 1 ? kTpFlagBytes + 2 * tp * ((N + tp - 1) / tp) * H * 4 : 0;  // peer-exchange arena
}

void Model::memory_bytes(int64_t out[5]) const {
    int64_t pf = 0;
    for (const auto& kv : params_) pf += 4 * kv.second.numel + (kv.second.bf ? 2 * kv.second.numel : 0);
    out[0] = pf;
    out[1] = 4 * grad_numel_;
    out[2] = (opt_m_ ? 4 * grad_numel_ : 0) + (opt_v_ ? 4 * grad_numel_ : 0);
    out[3] = static_cast<int64_t>(arena_.cap());
    out[4] = tpx_own_ ? tpx_bytes_ * (tp_virtual_ ? tp_ : 1) : 0;
}

// ------------------------------------------------------------------ tensor-parallel block
// Megatron head/column split: rank r owns heads [r nh/P, (r+1) nh/P) of the self- and cross-attention
// (its rows of the rank-major qkv / kv weights and of xattn.q, its entries of attn.temp) and rows
// [r 4H/P, (r+1) 4H/P) of ffn.in; attn.out / xattn.out / ffn.out are row-parallel (column blocks), so
// each residual branch ends in one exchange of an N x H fp32 partial.  Norms, gains, modulation and the
// heads are replicated.  Storage is partitioned: slot k (rank ranks[k]) has its own weight blocks
// (Ws / Ps / Gs) and its own compact activations of width H/P (qkv 3H/P, qk 2H/P, O / cqs / Ox H/P,
// kv 2H/P, z / h 4H/P); a real rank holds one slot, emulated ranks all P.
template <class T>
void Model::block_fwd_tp(int i, int64_t N) {
    WS& w = *ws_;
    const bool bf = bf16_;
    cudaStream_t s = stream_;
    const int64_t H = cfg_.H(), nh = cfg_.heads, hd = cfg_.hd(), L = w.L, td = cfg_.text_dim;
    const int64_t Hr = H / tp_, nhr = nh / tp_, Fr = 4 * H / tp_, lld = (N + 127) / 128 * 128;  // 128-row lse tiles
    Blk& b = w.blk[w.grads && !w.recompute ? i : 0];
    const float* Xin = w.X[w.grads ? i : (i % 2)];
    float* Xout = w.X[w.grads ? i + 1 : ((i + 1) % 2)];
    const float* tab = w.table[i];
    const int64_t tld = 6 * H;
    const int n = static_cast<int>(N);
    const std::vector<int> ranks = tp_ranks();
    auto acc = [&](size_t k) { return tp_virtual_ && k > 0 ? 1 : 0; };
    float* part = w.tpp;
    const float* sum = nullptr;
    // row-parallel GEMM: peer mode scatters the partial into the owners' mailboxes from the epilogue
    auto rowpar = [&](size_t k, int64_t r, const auto& A, const auto& B, int K, float alpha) {
        if (tp_peer_on())
            gemm(bf, A, B, n, int(H), K, tp_epi(tpx_base_, tp_, int(r), alpha, N, H, tpx_bf16_), s);
        else
            gemm(bf, A, B, n, int(H), K, EpiF32{part, H, nullptr, alpha, acc(k), n, int(H)}, s);
    };
    tp_peer_ensure(N);
    // self-attention (dit.cpp:287-297): column-parallel qkv, local heads, row-parallel out-proj
    rms_mod<T>(Xin, n, H, tab, tld, 0, H, w.mod_id, tp<T>(b.a), b.r0, s);
    for (size_t k = 0; k < ranks.size(); ++k) {
        const int64_t r = ranks[k];
        const int kk = static_cast<int>(k);
        void* qkv_r = off<T>(b.qkv, k * N * 3 * Hr);
        void* qk_r = off<T>(b.qk, k * N * 2 * Hr);
        void* O_r = off<T>(b.O, k * N * Hr);
        qkv_norm_rope<T>(bf, b.a, H, Ws(blk(i, "attn.qkv.w"), kk), Ps(blk(i, "attn.qkv.b"), kk), n, Hr, nhr,
                         QKLayout{3 * Hr, Hr, 2 * Hr, Hr, nh}, Ps(blk(i, "attn.temp"), kk), w.cs, qkv_r, qk_r,
                         b.iq + r * nhr, b.ik + r * nhr, s);
        AttnProblem ap{qk_r, 2 * Hr, off<T>(qk_r, Hr), 2 * Hr, off<T>(qkv_r, 2 * Hr), 3 * Hr, O_r, Hr,
                       b.lse + r * nhr * lld, n, n, int(nhr), int(hd)};
        ap.lse_ld = lld;
        ap.seg = w.seg;
        prof_.begin("attn_fwd", s);
        if (!w.recompute_pass) attention_fwd<T>(bf, ap, s);  // kept O / lse on recompute
        prof_.end(s);
        rowpar(k, r, KM(O_r, Hr), KM(Ws(blk(i, "attn.out.w"), kk), Hr), int(Hr), 1.0f);
    }
    sum = tp_exchange(part, N, s);
    bias_gate_resid<T>(sum, P(blk(i, "attn.out.b")).f32, tab, tld, int(2 * H), w.mod_id, Xin, b.X1, tp<T>(b.ao), n,
                       int(H), s);
    // cross-attention (dit.cpp:300-305)
    rms_gain<T>(b.X1, n, H, P(blk(i, "xattn.prenorm.g")).f32, tp<T>(b.cn), b.r1, s);
    const float xscale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(hd)));
    for (size_t k = 0; k < ranks.size(); ++k) {
        const int64_t r = ranks[k];
        const int kk = static_cast<int>(k);
        void* kv_r = off<T>(b.kv, k * L * 2 * Hr);
        void* cqs_r = off<T>(b.cqs, k * N * Hr);
        void* Ox_r = off<T>(b.Ox, k * N * Hr);
        gemm(bf, KM(b.cn, H), KM(Ws(blk(i, "xattn.q.w"), kk), H), n, int(Hr), H,
             EpiStore<T>{tp<T>(cqs_r), Hr, Ps(blk(i, "xattn.q.b"), kk), xscale, n, int(Hr)}, s);
        gemm(bf, KM(w.text, td), KM(Ws(blk(i, "xattn.kv.w"), kk), td), int(L), int(2 * Hr), td,
             EpiStore<T>{tp<T>(kv_r), 2 * Hr, Ps(blk(i, "xattn.kv.b"), kk), 1.0f, int(L), int(2 * Hr)}, s);
        AttnProblem xp{cqs_r, Hr, kv_r, 2 * Hr, off<T>(kv_r, Hr), 2 * Hr, Ox_r, Hr, b.lse_x + r * nhr * lld, n,
                       int(L), int(nhr), int(hd)};
        xp.lse_ld = lld;
        prof_.begin("xattn_fwd", s);
        attention_fwd<T>(bf, xp, s);
        prof_.end(s);
        rowpar(k, r, KM(Ox_r, Hr), KM(Ws(blk(i, "xattn.out.w"), kk), Hr), int(Hr), 1.0f);
    }
    sum = tp_exchange(part, N, s);
    bias_to<T>(sum, P(blk(i, "xattn.out.b")).f32, tp<T>(b.co), n, int(H), s);
    if (!(g_fusions & kFuseNormMod) ||
        !postnorm_resid_mod<T>(b.X1, tp<T>(b.co), n, H, P(blk(i, "xattn.postnorm.g")).f32, b.X2, b.rc, tab, tld,
                               3 * H, 4 * H, w.mod_id, tp<T>(b.f), b.r2, s)) {
        postnorm_resid<T>(b.X1, tp<T>(b.co), n, H, P(blk(i, "xattn.postnorm.g")).f32, b.X2, b.rc, s);
        rms_mod<T>(b.X2, n, H, tab, tld, 3 * H, 4 * H, w.mod_id, tp<T>(b.f), b.r2, s);
    }
    // feed-forward (dit.cpp:308-311): column-parallel ffn.in, row-parallel ffn.out
    for (size_t k = 0; k < ranks.size(); ++k) {
        const int64_t r = ranks[k];
        const int kk = static_cast<int>(k);
        void* z_r = off<T>(b.z, k * N * Fr);
        void* h_r = off<T>(b.h, k * N * Fr);
        gemm(bf, KM(b.f, H), KM(Ws(blk(i, "ffn.in.w"), kk), H), n, int(Fr), H,
             EpiBiasSilu<T>{tp<T>(z_r), tp<T>(h_r), Fr, Ps(blk(i, "ffn.in.b"), kk), n, int(Fr)}, s);
        rowpar(k, r, KM(h_r, Fr), KM(Ws(blk(i, "ffn.out.w"), kk), Fr), int(Fr), 1.0f);
    }
    sum = tp_exchange(part, N, s);
    bias_gate_resid<T>(sum, P(blk(i, "ffn.out.b")).f32, tab, tld, int(5 * H), w.mod_id, b.X2, Xout, tp<T>(b.ff), n,
                       int(H), s);
}

template <class T>
void Model::block_bwd_tp(int i, int64_t N) {
    WS& w = *ws_;
    const bool bf = bf16_;
    cudaStream_t s = stream_;
    const int64_t H = cfg_.H(), nh = cfg_.heads, hd = cfg_.hd(), L = w.L, td = cfg_.text_dim;
    const int64_t Hr = H / tp_, nhr = nh / tp_, Fr = 4 * H / tp_, lld = (N + 127) / 128 * 128;  // 128-row lse tiles
    const int n = static_cast<int>(N), nu = w.n_u, chunks = row_chunks(n);
    Blk& b = w.blk[w.recompute ? 0 : i];
    const float* Xin = w.X[i];
    const float* tab = w.table[i];
    const int64_t tld = 6 * H;
    float* dX = w.dX;
    float* dm = w.dm;
    const std::vector<int> ranks = tp_ranks();
    auto acc = [&](size_t k) { return tp_virtual_ && k > 0 ? 1 : 0; };
    float* part = w.tpp;
    const float* sum = nullptr;
    // row-parallel GEMM: peer mode scatters the partial into the owners' mailboxes from the epilogue
    auto rowpar = [&](size_t k, int64_t r, const auto& A, const auto& B, int K, float alpha) {
        if (tp_peer_on())
            gemm(bf, A, B, n, int(H), K, tp_epi(tpx_base_, tp_, int(r), alpha, N, H, tpx_bf16_), s);
        else
            gemm(bf, A, B, n, int(H), K, EpiF32{part, H, nullptr, alpha, acc(k), n, int(H)}, s);
    };
    tp_peer_ensure(N);
    // ---- FFN (dit.cpp:308-311)
    gate_bwd<T>(dX, tp<T>(b.ff), tab, tld, 5 * H, w.mod_id, nu, n, H, tp<T>(w.s1), w.part1, w.part2, s);
    reduce_chunks_grouped(w.part1, chunks, nu, H, dm + 5 * H, 6 * H, 1.0f, 0, s);  // d gt2
    reduce_chunks(w.part2, chunks, H, G(blk(i, "ffn.out.b")), 1.0f, 1, s);
    for (size_t k = 0; k < ranks.size(); ++k) {
        const int64_t r = ranks[k];
        const int kk = static_cast<int>(k);
        void* dz_r = off<T>(w.sA, k * N * Fr);
        gemm(bf, MN(w.s1, H), MN(off<T>(b.h, k * N * Fr), Fr), H, int(Fr), n,
             EpiF32{Gs(blk(i, "ffn.out.w"), kk), Fr, nullptr, 1.0f, 1, int(H), int(Fr)}, s);
        gemm(bf, KM(w.s1, H), MN(Ws(blk(i, "ffn.out.w"), kk), Fr), n, int(Fr), H,
             EpiSiluBwd<T>{tp<T>(dz_r), tp<T>(off<T>(b.z, k * N * Fr)), Fr, n, int(Fr)}, s);
        colsum<T>(tp<T>(dz_r), Fr, n, int(Fr), w.part1, s);
        reduce_chunks(w.part1, chunks, int(Fr), Gs(blk(i, "ffn.in.b"), kk), 1.0f, 1, s);
        gemm(bf, MN(dz_r, Fr), MN(b.f, H), int(Fr), H, n,
             EpiF32{Gs(blk(i, "ffn.in.w"), kk), H, nullptr, 1.0f, 1, int(Fr), int(H)}, s);
        rowpar(k, r, KM(dz_r, Fr), MN(Ws(blk(i, "ffn.in.w"), kk), H), int(Fr), 1.0f);  // df partial
    }
    sum = tp_exchange(part, N, s);
    convert_f32<T>(sum, N * H, tp<T>(w.s1), s);
    rms_mod_bwd<T>(tp<T>(w.s1), b.X2, b.r2, tab, tld, 3 * H, 4 * H, w.mod_id, nu, n, H, dX, w.part1, w.part2, s);
    reduce_chunks_grouped(w.part1, chunks, nu, H, dm + 3 * H, 6 * H, 1.0f, 0, s);  // d sh2
    reduce_chunks_grouped(w.part2, chunks, nu, H, dm + 4 * H, 6 * H, 1.0f, 0, s);  // d sc2
    // ---- cross-attention (dit.cpp:300-305)
    postnorm_bwd<T>(dX, tp<T>(b.co), b.rc, P(blk(i, "xattn.postnorm.g")).f32, n, H, tp<T>(w.s1), w.part1, s);
    reduce_chunks(w.part1, chunks, H, G(blk(i, "xattn.postnorm.g")), 1.0f, 1, s);
    colsum<T>(tp<T>(w.s1), H, n, H, w.part1, s);
    reduce_chunks(w.part1, chunks, H, G(blk(i, "xattn.out.b")), 1.0f, 1, s);
    for (size_t k = 0; k < ranks.size(); ++k) {  // all slots read the full dco (s1) before their dq overwrites it
        const int kk = static_cast<int>(k);
        gemm(bf, MN(w.s1, H), MN(off<T>(b.Ox, k * N * Hr), Hr), H, int(Hr), n,
             EpiF32{Gs(blk(i, "xattn.out.w"), kk), Hr, nullptr, 1.0f, 1, int(H), int(Hr)}, s);
        gemm(bf, KM(w.s1, H), MN(Ws(blk(i, "xattn.out.w"), kk), Hr), n, int(Hr), H,
             EpiStore<T>{tp<T>(off<T>(w.s2, k * N * Hr)), Hr, nullptr, 1.0f, n, int(Hr)}, s);
    }
    const float xscale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(hd)));
    for (size_t k = 0; k < ranks.size(); ++k) {
        const int64_t r = ranks[k];
        const int kk = static_cast<int>(k);
        void* kv_r = off<T>(b.kv, k * L * 2 * Hr);
        void* dkv_r = off<T>(w.dkv, k * L * 2 * Hr);
        void* dq_r = off<T>(w.s1, k * N * Hr);
        AttnBwdProblem xb{AttnProblem{off<T>(b.cqs, k * N * Hr), Hr, kv_r, 2 * Hr, off<T>(kv_r, Hr), 2 * Hr,
                                      off<T>(b.Ox, k * N * Hr), Hr, b.lse_x + r * nhr * lld, n, int(L), int(nhr),
                                      int(hd)},
                          off<T>(w.s2, k * N * Hr), Hr, w.Dvec + r * nhr * lld, dq_r, Hr, dkv_r, 2 * Hr,
                          off<T>(dkv_r, Hr), 2 * Hr, w.dkv_part + r * (int64_t)w.q_splits_x * nhr * L * 2 * hd,
                          w.q_splits_x};
        xb.f.lse_ld = lld;
        prof_.begin("xattn_bwd", s);
        attention_bwd<T>(bf, xb, s);
        prof_.end(s);
        gemm(bf, MN(dkv_r, 2 * Hr), MN(w.text, td), int(2 * Hr), td, int(L),
             EpiF32{Gs(blk(i, "xattn.kv.w"), kk), td, nullptr, 1.0f, 1, int(2 * Hr), int(td)}, s);
        colsum<T>(tp<T>(dkv_r), 2 * Hr, int(L), int(2 * Hr), w.part1, s);
        reduce_chunks(w.part1, row_chunks(int(L)), int(2 * Hr), Gs(blk(i, "xattn.kv.b"), kk), 1.0f, 1, s);
        colsum<T>(tp<T>(dq_r), Hr, n, int(Hr), w.part1, s);
        reduce_chunks(w.part1, chunks, int(Hr), Gs(blk(i, "xattn.q.b"), kk), xscale, 1, s);
        gemm(bf, MN(dq_r, Hr), MN(b.cn, H), int(Hr), H, n,
             EpiF32{Gs(blk(i, "xattn.q.w"), kk), H, nullptr, xscale, 1, int(Hr), int(H)}, s);
        rowpar(k, r, KM(dq_r, Hr), MN(Ws(blk(i, "xattn.q.w"), kk), H), int(Hr), xscale);  // dcn partial
    }
    sum = tp_exchange(part, N, s);
    convert_f32<T>(sum, N * H, tp<T>(w.s2), s);
    rms_gain_bwd<T>(tp<T>(w.s2), b.X1, b.r1, P(blk(i, "xattn.prenorm.g")).f32, n, H, dX, 1, w.part1, s);
    reduce_chunks(w.part1, chunks, H, G(blk(i, "xattn.prenorm.g")), 1.0f, 1, s);
    // ---- self-attention (dit.cpp:287-297)
    gate_bwd<T>(dX, tp<T>(b.ao), tab, tld, 2 * H, w.mod_id, nu, n, H, tp<T>(w.s1), w.part1, w.part2, s);
    reduce_chunks_grouped(w.part1, chunks, nu, H, dm + 2 * H, 6 * H, 1.0f, 0, s);  // d gt1
    reduce_chunks(w.part2, chunks, H, G(blk(i, "attn.out.b")), 1.0f, 1, s);
    for (size_t k = 0; k < ranks.size(); ++k) {
        const int kk = static_cast<int>(k);
        gemm(bf, MN(w.s1, H), MN(off<T>(b.O, k * N * Hr), Hr), H, int(Hr), n,
             EpiF32{Gs(blk(i, "attn.out.w"), kk), Hr, nullptr, 1.0f, 1, int(H), int(Hr)}, s);
        gemm(bf, KM(w.s1, H), MN(Ws(blk(i, "attn.out.w"), kk), Hr), n, int(Hr), H,
             EpiStore<T>{tp<T>(off<T>(w.s2, k * N * Hr)), Hr, nullptr, 1.0f, n, int(Hr)}, s);
    }
    for (size_t k = 0; k < ranks.size(); ++k) {
        const int64_t r = ranks[k];
        const int kk = static_cast<int>(k);
        void* qkv_r = off<T>(b.qkv, k * N * 3 * Hr);
        void* qk_r = off<T>(b.qk, k * N * 2 * Hr);
        void* dqkv_r = off<T>(w.sB, k * N * 3 * Hr);
        AttnBwdProblem ab{AttnProblem{qk_r, 2 * Hr, off<T>(qk_r, Hr), 2 * Hr, off<T>(qkv_r, 2 * Hr), 3 * Hr,
                                      off<T>(b.O, k * N * Hr), Hr, b.lse + r * nhr * lld, n, n, int(nhr), int(hd)},
                          off<T>(w.s2, k * N * Hr), Hr, w.Dvec + r * nhr * lld, dqkv_r, 3 * Hr, off<T>(dqkv_r, Hr),
                          3 * Hr, off<T>(dqkv_r, 2 * Hr), 3 * Hr, nullptr, 1};
        ab.f.lse_ld = lld;
        ab.f.seg = w.seg;
        prof_.begin("attn_bwd", s);
        attention_bwd<T>(bf, ab, s);
        prof_.end(s);
        qk_norm_rope_bwd<T>(tp<T>(dqkv_r), tp<T>(qkv_r), QKLayout{3 * Hr, Hr, 2 * Hr, Hr, nh}, n, int(Hr), int(nhr),
                            Ps(blk(i, "attn.temp"), kk), w.cs, b.iq + r * nhr, b.ik + r * nhr, w.part1, s);
        reduce_chunks(w.part1, chunks, int(nhr), Gs(blk(i, "attn.temp"), kk), 1.0f, 1, s);
        colsum<T>(tp<T>(dqkv_r), 3 * Hr, n, int(3 * Hr), w.part1, s);
        reduce_chunks(w.part1, chunks, int(3 * Hr), Gs(blk(i, "attn.qkv.b"), kk), 1.0f, 1, s);
        gemm(bf, MN(dqkv_r, 3 * Hr), MN(b.a, H), int(3 * Hr), H, n,
             EpiF32{Gs(blk(i, "attn.qkv.w"), kk), H, nullptr, 1.0f, 1, int(3 * Hr), int(H)}, s);
        rowpar(k, r, KM(dqkv_r, 3 * Hr), MN(Ws(blk(i, "attn.qkv.w"), kk), H), int(3 * Hr), 1.0f);  // da partial
    }
    sum = tp_exchange(part, N, s);
    convert_f32<T>(sum, N * H, tp<T>(w.s1), s);
    rms_mod_bwd<T>(tp<T>(w.s1), Xin, b.r0, tab, tld, 0, H, w.mod_id, nu, n, H, dX, w.part1, w.part2, s);
    reduce_chunks_grouped(w.part1, chunks, nu, H, dm, 6 * H, 1.0f, 0, s);      // d sh1
    reduce_chunks_grouped(w.part2, chunks, nu, H, dm + H, 6 * H, 1.0f, 0, s);  // d sc1
    // ---- shared modulation head (dit.cpp:280-283), replicated
    modulation_bwd(dm, w.gb[i], P("dit.mod.w").f32, nu, H, G("dit.mod.w"), G("dit.mod.b"), w.dgb, s);
    gscale_bwd(w.dgb, w.g, P(blk(i, "gscale")).f32, nu, H, G(blk(i, "gscale")), w.dg, s);
}

// ------------------------------------------------------------------ sample forward / backward
// rows_in: (N, D) T on device (for velocity) or null with X[0] preloaded (dit_forward).
template <class T>
void Model::forward_sample(const DevSample& smp, const void* rows_in, const double* taus_unique, int n_u,
                           const int32_t* mod_id, double fps, bool grads, bool head, void* out) {
    (void)smp;
    (void)taus_unique;
    (void)mod_id;
    (void)out;
    WS& w = *ws_;
    cudaStream_t s = stream_;
    const bool bf = bf16_;
    const int64_t H = cfg_.H(), D = cfg_.D();
    const int n = static_cast<int>(w.N);
    // global embedding + per-block modulation tables over the n_u unique timesteps (dit.cpp:236-255, 280-283)
    global_embed(w.taus, n_u, fps, P("dit.gmlp.in.w").f32, P("dit.gmlp.in.b").f32, P("dit.gmlp.out.w").f32,
                 P("dit.gmlp.out.b").f32, H, w.phi, w.z_in, w.h_in, w.g, s);
    for (int i = 0; i < cfg_.depth; ++i)
        modulation_table(w.g, P(blk(i, "gscale")).f32, P("dit.mod.w").f32, P("dit.mod.b").f32, n_u, H, w.gb[i],
                         w.table[i], s);
    rope_table(w.coords, n, cfg_.rope[0], cfg_.rope[1], cfg_.rope[2], w.cs, s);
    if (head)  // patch embedding (dit.cpp:327)
        gemm(bf, KM(rows_in, D), KM(W("dit.patch.w"), D), n, H, D,
             EpiF32{w.X[0], H, P("dit.patch.b").f32, 1.0f, 0, n, int(H)}, s);
    (void)grads;
    prof_.begin("blocks_fwd", s);
    for (int i = 0; i < cfg_.depth; ++i) {
        use_block_slot(i);
        block_fwd<T>(i, w.N);
    }
    prof_.end(s);
    const float* Xf = w.X[w.grads ? cfg_.depth : (cfg_.depth % 2)];
    rms_gain<T>(Xf, n, H, P("dit.final.g").f32, tp<T>(w.fin), w.rf, s);  // dit.cpp:314
    if (head) {
        gemm(bf, KM(w.fin, H), KM(W("dit.final.w"), H), n, H, H,
             EpiStore<T>{tp<T>(w.Y), H, P("dit.final.b").f32, 1.0f, n, int(H)}, s);  // dit.cpp:315
        gemm(bf, KM(w.Y, H), KM(W("dit.out.w"), H), n, D, H, EpiF32{w.V, D, P("dit.out.b").f32, 1.0f, 0, n, int(D)},
             s);  // dit.cpp:331
    } else {
        gemm(bf, KM(w.fin, H), KM(W("dit.final.w"), H), n, H, H,
             EpiF32{static_cast<float*>(out), H, P("dit.final.b").f32, 1.0f, 0, n, int(H)}, s);
    }
}

template <class T>
void Model::backward_sample(const void* dV) {
    WS& w = *ws_;
    cudaStream_t s = stream_;
    const bool bf = bf16_;
    const int64_t H = cfg_.H(), D = cfg_.D();
    const int n = static_cast<int>(w.N), chunks = row_chunks(n), nu = w.n_u;
    // heads (dit.cpp:331, 314-315)
    gemm(bf, MN(dV, D), MN(w.Y, H), int(D), H, n, EpiF32{G("dit.out.w"), H, nullptr, 1.0f, 1, int(D), int(H)}, s);
    colsum<T>(tp<T>(dV), D, n, D, w.part1, s);
    reduce_chunks(w.part1, chunks, D, G("dit.out.b"), 1.0f, 1, s);
    gemm(bf, KM(dV, D), MN(W("dit.out.w"), H), n, H, D, EpiStore<T>{tp<T>(w.s1), H, nullptr, 1.0f, n, int(H)}, s);
    gemm(bf, MN(w.s1, H), MN(w.fin, H), H, H, n, EpiF32{G("dit.final.w"), H, nullptr, 1.0f, 1, int(H), int(H)}, s);
    colsum<T>(tp<T>(w.s1), H, n, H, w.part1, s);
    reduce_chunks(w.part1, chunks, H, G("dit.final.b"), 1.0f, 1, s);
    gemm(bf, KM(w.s1, H), MN(W("dit.final.w"), H), n, H, H, EpiStore<T>{tp<T>(w.s2), H, nullptr, 1.0f, n, int(H)}, s);
    rms_gain_bwd<T>(tp<T>(w.s2), w.X[cfg_.depth], w.rf, P("dit.final.g").f32, n, H, w.dX, 0, w.part1, s);
    reduce_chunks(w.part1, chunks, H, G("dit.final.g"), 1.0f, 1, s);
    MGV_CUDA(cudaMemsetAsync(w.dg, 0, sizeof(double) * nu * H, s));
    prof_.begin("blocks_bwd", s);
    for (int i = static_cast<int>(cfg_.depth) - 1; i >= 0; --i) {
        // per-block recompute: slot 0 holds the last block's activations after the forward; every other block's
        // are rebuilt from its kept input X[i] (same kernels, same inputs: bit-identical to keeping them)
        use_block_slot(i);
        if (w.recompute && i + 1 < cfg_.depth) {
            prof_.begin("recompute", s);
            w.recompute_pass = true;
            block_fwd<T>(i, w.N);
            w.recompute_pass = false;
            prof_.end(s);
        }
        block_bwd<T>(i, w.N);
    }
    prof_.end(s);
    // patch embedding (rows are constants, dit.cpp:327)
    convert_f32<T>(w.dX, (int64_t)n * H, tp<T>(w.s1), s);
    gemm(bf, MN(w.s1, H), MN(w.rows, D), H, int(D), n, EpiF32{G("dit.patch.w"), D, nullptr, 1.0f, 1, int(H), int(D)}, s);
    colsum<float>(w.dX, H, n, H, w.part1, s);
    reduce_chunks(w.part1, chunks, H, G("dit.patch.b"), 1.0f, 1, s);
    // global embedding MLPs (dit.cpp:245-254)
    global_embed_bwd(w.dg, nu, w.phi, w.z_in, w.h_in, P("dit.gmlp.out.w").f32, H, G("dit.gmlp.in.w"),
                     G("dit.gmlp.in.b"), G("dit.gmlp.out.w"), G("dit.gmlp.out.b"), s);
}

// ------------------------------------------------------------------ flow step
static double wk_of(const StepExtra* ex, int64_t k, int64_t B) {
    return ex && ex->weight ? ex->weight[k] : 1.0 / static_cast<double>(B);
}

// AdamW::update (optim.cpp:7-24) over every parameter slot held here; the kernel skips the update when the step's
// loss accumulator is not finite (FlowTrainer::step throws before updating, flowtrain.cpp:276)
void Model::adamw_step(cudaStream_t s) {
    WS& w = *ws_;
    if (!opt_m_) alloc_adam_state();
    ++adam_.step;
    const double bc1 = 1.0 - std::pow(adam_.b1, static_cast<double>(adam_.step));
    const double bc2 = 1.0 - std::pow(adam_.b2, static_cast<double>(adam_.step));
    int64_t maxn = 0;
    for (auto* q : sorted_) maxn = std::max(maxn, q->numel);
    const dim3 grid(static_cast<unsigned>(std::min<int64_t>((maxn / 4 + 255) / 256, 592)),
                    static_cast<unsigned>(sorted_.size()));
    prof_.begin("adamw", s);
    adamw_kernel<<<grid, 256, 0, s>>>(static_cast<const AdamParam*>(param_table_), grad_buf_, opt_m_, opt_v_, w.scal,
                                      float(adam_.lr), float(adam_.b1), float(adam_.b2), float(adam_.eps),
                                      float(adam_.wd), float(1.0 / bc1), float(1.0 / bc2));
    note_launch();
    MGV_CUDA(cudaGetLastError());
    prof_.end(s);
}

template <class T>
void Model::flow_step_impl(int64_t n, const DevSample* samples, const double* text_dev, int64_t L, double fps,
                           double* loss, double* grad_norm, double* const* v_dev, const StepExtra* ex) {
    if (!have_params_) throw InputError("no parameters uploaded");
    if (n < 1) throw InputError("empty batch");  // flowtrain.cpp:258
    WS& w = *ws_;
    cudaStream_t s = stream_;
    const int64_t D = cfg_.D();
    int64_t maxN = 0;
    for (int64_t k = 0; k < n; ++k) maxN = std::max(maxN, samples[k].N);
    const bool per_text = ex && ex->text_dev;
    const bool backward = !ex || ex->backward;
    if (ex && world_ > 1) throw ConfigError("weighted / forward-only steps run without data parallelism");
    int64_t maxL = L;
    if (per_text)
        for (int64_t k = 0; k < n; ++k) maxL = std::max(maxL, ex->L[k]);
    // workspace (arena grows only; the layout is re-derived for this batch)
    w.N = maxN;
    w.L = maxL;
    w.n_u = 2;
    w.esz = bf16_ ? 2 : 4;
    w.grads = true;
    w.tp = tp_;
    w.tp_slots = tp_slots();
    w.recompute = recompute_ && w.grads;
    set_tpose(w, cfg_);
    {
        Sizer sz{true, 0, &arena_};
        layout_ws(w, sz, cfg_, true);
        arena_.reserve(sz.bytes);
        arena_.reset();
        Sizer real{false, 0, &arena_};
        layout_ws(w, real, cfg_, true);
    }
    const int64_t launches0 = launch_count();
    cudaEvent_t e0, e1;
    MGV_CUDA(cudaEventCreate(&e0));
    MGV_CUDA(cudaEventCreate(&e1));
    MGV_CUDA(cudaEventRecord(e0, s));
    prof_.begin_step();
    GemmProfGuard gemm_prof(prof_);
    MGV_CUDA(cudaMemsetAsync(grad_buf_, 0, sizeof(float) * grad_numel_, s));
    MGV_CUDA(cudaMemsetAsync(w.scal, 0, sizeof(double) * 8, s));
    if (!per_text) convert_rows<T>(text_dev, L * cfg_.text_dim, tp<T>(w.text), s);
    const int64_t B_global = n * world_;
    std::vector<double> errs_host(static_cast<size_t>(ex ? n : 0));
    double* errs_dev = nullptr;  // l_k per sample (weighted / forward-only steps)
    if (ex) {
        MGV_CUDA(cudaMallocAsync(&errs_dev, sizeof(double) * n, s));
        MGV_CUDA(cudaMemsetAsync(errs_dev, 0, sizeof(double) * n, s));
    }
    const double* prev_text = nullptr;
    for (int64_t k = 0; k < n; ++k) {
        const DevSample& sm = samples[k];
        w.N = sm.N;
        if (per_text) {  // this record's text (converted once per distinct pointer)
            w.L = ex->L[k];
            if (ex->text_dev[k] != prev_text)
                convert_rows<T>(ex->text_dev[k], ex->L[k] * cfg_.text_dim, tp<T>(w.text), s);
            prev_text = ex->text_dev[k];
        }
        const double fps_k = ex && ex->fps ? ex->fps[k] : fps;
        const double wk = ex && ex->weight ? ex->weight[k] : 1.0 / static_cast<double>(B_global);
        const int N = static_cast<int>(sm.N);
        MGV_CUDA(cudaMemcpyAsync(w.coords, sm.coords, sizeof(int32_t) * 3 * N, cudaMemcpyDeviceToDevice, s));
        // interpolate + condition mask (flowtrain.cpp:265-267); taus {t, 0} (dit.cpp:242 dedup)
        prep_flow_sample<T>(sm.clean, sm.noise, sm.cond, sm.cond_lat, N, int(D), sm.t, tp<T>(w.rows), w.vt, w.lmask,
                            w.mod_id, s);
        w.n_u = sm.cond ? 2 : 1;
        set_taus(w.taus, sm.t, s);
        forward_sample<T>(sm, w.rows, nullptr, w.n_u, w.mod_id, fps_k, true, true, nullptr);
        if (v_dev && v_dev[k]) {
            f32_to_f64<<<grid_of(N * D), 256, 0, s>>>(w.V, N * D, v_dev[k]);
            note_launch();
        }
        // masked mean loss (autodiff.cpp:466-491), coefficient and accumulation on device
        count_mask(w.lmask, N, w.cnt, s);
        flow_loss_fwd<T>(w.V, w.vt, w.lmask, N, int(D), w.loss_part, s);
        flow_loss_accumulate(w.loss_part, row_chunks(N), w.cnt, int(D), w.scal, s);  // scal[0] += l_b
        if (ex) flow_loss_accumulate(w.loss_part, row_chunks(N), w.cnt, int(D), errs_dev + k, s);  // l_k alone
        if (backward && wk != 0.0) {
            flow_loss_bwd<T>(w.V, w.vt, w.lmask, N, int(D), static_cast<float>(2.0 * wk), w.cnt, tp<T>(w.dV),
                             s);  // 2 w_k (V - v*) / (n_b * D), w_k = 1 / B in FlowTrainer::step; all-masked -> 0
            // per-block buckets need each block's gradients contiguous: sorted names, i.e. no TP layout
            dp_overlap_ = comm_ != nullptr && !ex && k == n - 1 && tp_ == 1;
            dp_done_.clear();
            backward_sample<T>(w.dV);
            dp_overlap_ = false;
        }
    }
    if (ex) {
        MGV_CUDA(cudaMemcpyAsync(errs_host.data(), errs_dev, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
        MGV_CUDA(cudaFreeAsync(errs_dev, s));
    }
    if (!backward) {  // flow errors only
        double host2 = 0.0;
        MGV_CUDA(cudaStreamSynchronize(s));
        last_launches_ = launch_count() - launches0;
        prof_.end_step();
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        for (int64_t k = 0; k < n; ++k) {
            ex->errs[k] = errs_host[static_cast<size_t>(k)];
            host2 += (ex->weight ? ex->weight[k] : 1.0 / static_cast<double>(B_global)) * ex->errs[k];
        }
        *loss = host2;
        if (grad_norm) *grad_norm = 0.0;
        return;
    }
    tp_allreduce_grads(s);
    if (comm_) {
        prof_.begin("allreduce", s);
        dp_finish(w.scal);
        prof_.end(s);
    }
    // grad_norm (flowtrain.cpp:284-289); under TP the sharded blocks' squares are summed over the TP group
    if (tp_ > 1) {
        sumsq(grad_buf_, repl_numel_, w.loss_part, w.scal + 2, s);
        sumsq(grad_buf_ + repl_numel_, grad_numel_ - repl_numel_, w.loss_part, w.scal + 3, s);
        if (!tp_virtual_) MGV_NCCL(ncclAllReduce(w.scal + 3, w.scal + 3, 1, ncclDouble, ncclSum, tp_comm_, s));
    } else {
        sumsq(grad_buf_, grad_numel_, w.loss_part, w.scal + 2, s);
    }
    if (adam_.on) adamw_step(s);  // AdamW::update (flowtrain.cpp:278), on device, skipped if the loss is not finite
    double host[4] = {0, 0, 0, 0};
    MGV_CUDA(cudaMemcpyAsync(host, w.scal, sizeof(double) * 4, cudaMemcpyDeviceToHost, s));
    MGV_CUDA(cudaEventRecord(e1, s));
    MGV_CUDA(cudaStreamSynchronize(s));
    check_comms();
    float ms = 0.0f;
    MGV_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    last_ms_ = ms;
    last_launches_ = launch_count() - launches0;
    prof_.end_step();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *loss = host[0] / static_cast<double>(B_global);  // flowtrain.cpp:273
    if (ex) {  // weighted: Loss = sum_k w_k l_k
        double tot = 0.0;
        for (int64_t k = 0; k < n; ++k) {
            if (ex->errs) ex->errs[k] = errs_host[static_cast<size_t>(k)];
            tot += wk_of(ex, k, B_global) * errs_host[static_cast<size_t>(k)];
        }
        *loss = tot;
    }
    if (!std::isfinite(*loss)) {  // flowtrain.cpp:276 (the device AdamW step was skipped)
        if (adam_.on) --adam_.step;
        throw NumericError("flow loss is not finite");
    }
    *grad_norm = std::sqrt(host[2] + (tp_ > 1 ? host[3] : 0.0));
}

void Model::flow_step_dev(int64_t n, const DevSample* samples, const double* text_dev, int64_t L, double fps,
                          double* loss, double* grad_norm, double* const* v_dev, const StepExtra* ex) {
    MGV_CUDA(cudaSetDevice(device_));
    const bool packed = varlen_ && n > 1 && !ex;
    if (bf16_)
        packed ? flow_step_packed<__nv_bfloat16>(n, samples, text_dev, L, fps, loss, grad_norm, v_dev)
               : flow_step_impl<__nv_bfloat16>(n, samples, text_dev, L, fps, loss, grad_norm, v_dev, ex);
    else
        packed ? flow_step_packed<float>(n, samples, text_dev, L, fps, loss, grad_norm, v_dev)
               : flow_step_impl<float>(n, samples, text_dev, L, fps, loss, grad_norm, v_dev, ex);
}

// Varlen packing (BASELINE configs[4]): the batch as ONE sequence of 256-row-aligned segments, one forward and
// one backward over all of it.  Attention is block-diagonal (AttnProblem::seg: each tile sees exactly its own
// sample's keys, with the step boundaries it has alone), the modulation table holds every sample's timestep plus
// 0 (mod_id per token), the RoPE table follows each token's coords, and the loss is each sample's masked mean over
// its own rows (flowtrain.cpp:263-273).  Padding rows are zero inputs with loss mask 0 and are never attended to,
// so every sample's forward is bit-identical to running it alone (dit_forward_batch's contract,
// test_dit.cpp:205-222); the gradients differ from per-sample accumulation only in summation order.
template <class T>
void Model::flow_step_packed(int64_t n, const DevSample* samples, const double* text_dev, int64_t L, double fps,
                             double* loss, double* grad_norm, double* const* v_dev) {
    if (!have_params_) throw InputError("no parameters uploaded");
    WS& w = *ws_;
    cudaStream_t s = stream_;
    const int64_t D = cfg_.D();
    std::vector<int64_t> base(static_cast<size_t>(n) + 1, 0);
    for (int64_t k = 0; k < n; ++k) base[k + 1] = base[k] + (samples[k].N + 255) / 256 * 256;
    const int64_t Np = base[n];
    w.N = Np;
    w.L = L;
    w.n_u = static_cast<int>(n) + 1;
    w.esz = bf16_ ? 2 : 4;
    w.grads = true;
    w.tp = tp_;
    w.tp_slots = tp_slots();
    w.recompute = recompute_ && w.grads;
    set_tpose(w, cfg_);
    {
        Sizer sz{true, 0, &arena_};
        layout_ws(w, sz, cfg_, true);
        arena_.reserve(sz.bytes);
        arena_.reset();
        Sizer real{false, 0, &arena_};
        layout_ws(w, real, cfg_, true);
    }
    const int64_t launches0 = launch_count();
    cudaEvent_t e0, e1;
    MGV_CUDA(cudaEventCreate(&e0));
    MGV_CUDA(cudaEventCreate(&e1));
    MGV_CUDA(cudaEventRecord(e0, s));
    prof_.begin_step();
    GemmProfGuard gemm_prof(prof_);
    MGV_CUDA(cudaMemsetAsync(grad_buf_, 0, sizeof(float) * grad_numel_, s));
    MGV_CUDA(cudaMemsetAsync(w.scal, 0, sizeof(double) * 8, s));
    convert_rows<T>(text_dev, L * cfg_.text_dim, tp<T>(w.text), s);
    // padding rows: zero inputs, zero targets, loss mask 0, coords (0, 0, 0), table row 0
    MGV_CUDA(cudaMemsetAsync(w.rows, 0, static_cast<size_t>(w.esz) * Np * D, s));
    MGV_CUDA(cudaMemsetAsync(w.vt, 0, sizeof(float) * Np * D, s));
    MGV_CUDA(cudaMemsetAsync(w.lmask, 0, Np, s));
    MGV_CUDA(cudaMemsetAsync(w.mod_id, 0, sizeof(int32_t) * Np, s));
    MGV_CUDA(cudaMemsetAsync(w.coords, 0, sizeof(int32_t) * 3 * Np, s));
    std::vector<double> taus(static_cast<size_t>(n) + 1, 0.0);  // t_0 .. t_{n-1}, then 0 (conditioned tokens)
    std::vector<int> seg(static_cast<size_t>(2 * ((Np + 127) / 128)));
    for (int64_t k = 0; k < n; ++k) {
        const DevSample& sm = samples[k];
        taus[static_cast<size_t>(k)] = sm.t;
        MGV_CUDA(cudaMemcpyAsync(w.coords + 3 * base[k], sm.coords, sizeof(int32_t) * 3 * sm.N, cudaMemcpyDeviceToDevice,
                                 s));
        if (base[k + 1] > base[k] + sm.N)  // padding rows: this sample's tau = t row (<= 2 rows per 64-row chunk)
            fill_i32(w.mod_id + base[k] + sm.N, base[k + 1] - base[k] - sm.N, static_cast<int>(k), s);
        prep_flow_sample<T>(sm.clean, sm.noise, sm.cond, sm.cond_lat, static_cast<int>(sm.N), int(D), sm.t,
                            tp<T>(off<T>(w.rows, base[k] * D)), w.vt + base[k] * D, w.lmask + base[k],
                            w.mod_id + base[k], s, static_cast<int>(k), static_cast<int>(n));
        for (int64_t t = base[k] / 128; t < base[k + 1] / 128; ++t) {
            seg[static_cast<size_t>(2 * t)] = static_cast<int>(base[k]);
            seg[static_cast<size_t>(2 * t + 1)] = static_cast<int>(base[k] + sm.N);
        }
    }
    MGV_CUDA(cudaMemcpyAsync(w.taus, taus.data(), sizeof(double) * taus.size(), cudaMemcpyHostToDevice, s));
    MGV_CUDA(cudaMemcpyAsync(w.segbuf, seg.data(), sizeof(int) * seg.size(), cudaMemcpyHostToDevice, s));
    w.seg = w.segbuf;
    DevSample dummy;
    forward_sample<T>(dummy, w.rows, nullptr, w.n_u, nullptr, fps, true, true, nullptr);
    const int64_t B_global = n * world_;
    MGV_CUDA(cudaMemsetAsync(w.dV, 0, static_cast<size_t>(w.esz) * Np * D, s));
    for (int64_t k = 0; k < n; ++k) {  // each sample's masked mean (autodiff.cpp:466-491) and its dV rows
        const int Nk = static_cast<int>(samples[k].N);
        const float* Vk = w.V + base[k] * D;
        if (v_dev && v_dev[k]) {
            f32_to_f64<<<grid_of(Nk * D), 256, 0, s>>>(Vk, Nk * D, v_dev[k]);
            note_launch();
        }
        count_mask(w.lmask + base[k], Nk, w.cnt, s);
        flow_loss_fwd<T>(Vk, w.vt + base[k] * D, w.lmask + base[k], Nk, int(D), w.loss_part, s);
        flow_loss_accumulate(w.loss_part, row_chunks(Nk), w.cnt, int(D), w.scal, s);
        flow_loss_bwd<T>(Vk, w.vt + base[k] * D, w.lmask + base[k], Nk, int(D),
                         static_cast<float>(2.0 / static_cast<double>(B_global)), w.cnt,
                         tp<T>(off<T>(w.dV, base[k] * D)), s);
    }
    dp_overlap_ = comm_ != nullptr && tp_ == 1;
    dp_done_.clear();
    backward_sample<T>(w.dV);
    dp_overlap_ = false;
    w.seg = nullptr;
    tp_allreduce_grads(s);
    if (comm_) {
        prof_.begin("allreduce", s);
        dp_finish(w.scal);
        prof_.end(s);
    }
    if (tp_ > 1) {
        sumsq(grad_buf_, repl_numel_, w.loss_part, w.scal + 2, s);
        sumsq(grad_buf_ + repl_numel_, grad_numel_ - repl_numel_, w.loss_part, w.scal + 3, s);
        if (!tp_virtual_) MGV_NCCL(ncclAllReduce(w.scal + 3, w.scal + 3, 1, ncclDouble, ncclSum, tp_comm_, s));
    } else {
        sumsq(grad_buf_, grad_numel_, w.loss_part, w.scal + 2, s);
    }
    if (adam_.on) adamw_step(s);
    double host[4] = {0, 0, 0, 0};
    MGV_CUDA(cudaMemcpyAsync(host, w.scal, sizeof(double) * 4, cudaMemcpyDeviceToHost, s));
    MGV_CUDA(cudaEventRecord(e1, s));
    MGV_CUDA(cudaStreamSynchronize(s));
    check_comms();
    float ms = 0.0f;
    MGV_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    last_ms_ = ms;
    last_launches_ = launch_count() - launches0;
    prof_.end_step();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *loss = host[0] / static_cast<double>(B_global);  // flowtrain.cpp:273
    if (!std::isfinite(*loss)) {  // flowtrain.cpp:276 (the device AdamW step was skipped)
        if (adam_.on) --adam_.step;
        throw NumericError("flow loss is not finite");
    }
    *grad_norm = std::sqrt(host[2] + (tp_ > 1 ? host[3] : 0.0));
}

// host-buffer flow step: validate, stage to device, run, read back
static void validate_mask_host(const mgv_flow_sample& s, int64_t N) {  // flowtrain.cpp:61-81
    if (!s.conditioned) return;
    std::vector<int> unit(static_cast<size_t>(s.dims[0]), -1);
    for (int64_t i = 0; i < N; ++i) {
        const int u = s.coords[3 * i];
        if (u < 0 || u >= s.dims[0]) throw DimensionError("condition mask does not match the token grid");
        const int f = s.conditioned[i] ? 1 : 0;
        int& seen = unit[static_cast<size_t>(u)];
        if (seen == -1)
            seen = f;
        else if (seen != f)
            throw InputError("conditioned tokens must cover whole latent units");
    }
}

// stage host samples on the device (validated as FlowTrainer::step / apply_condition_mask do)
void Model::stage_samples(int64_t n, const mgv_flow_sample* samples, std::vector<DevSample>& ds,
                          std::vector<void*>& allocs) {
    const int64_t D = cfg_.D();
    auto dalloc = [&](size_t bytes) {
        void* p = nullptr;
        MGV_CUDA(cudaMallocAsync(&p, bytes, stream_));
        allocs.push_back(p);
        return p;
    };
    ds.assign(static_cast<size_t>(n), DevSample{});
    for (int64_t k = 0; k < n; ++k) {
        const mgv_flow_sample& s = samples[k];
        const int64_t N = s.dims[0] * s.dims[1] * s.dims[2];
        if (N < 1) throw DimensionError("empty token grid");
        if (!s.coords || !s.clean_rows || !s.noise) throw InputError("null sample buffer");
        if (!(s.t >= 0.0 && s.t <= 1.0)) throw InputError("interpolation time outside [0, 1]");  // flowtrain.cpp:11
        validate_mask_host(s, N);
        bool cond_any = false;
        if (s.conditioned)
            for (int64_t i = 0; i < N && !cond_any; ++i) cond_any = s.conditioned[i] != 0;
        DevSample d;
        d.N = N;
        std::memcpy(d.dims, s.dims, sizeof(d.dims));
        auto* c = static_cast<int32_t*>(dalloc(sizeof(int32_t) * 3 * N));
        MGV_CUDA(cudaMemcpyAsync(c, s.coords, sizeof(int32_t) * 3 * N, cudaMemcpyHostToDevice, stream_));
        auto* cl = static_cast<double*>(dalloc(sizeof(double) * N * D));
        auto* nz = static_cast<double*>(dalloc(sizeof(double) * N * D));
        MGV_CUDA(cudaMemcpyAsync(cl, s.clean_rows, sizeof(double) * N * D, cudaMemcpyHostToDevice, stream_));
        MGV_CUDA(cudaMemcpyAsync(nz, s.noise, sizeof(double) * N * D, cudaMemcpyHostToDevice, stream_));
        d.coords = c;
        d.clean = cl;
        d.noise = nz;
        d.t = s.t;
        if (cond_any) {
            // apply_condition_mask (flowtrain.cpp:83-100): any unit-aligned mask; validate_mask requires the
            // condition latents (flowtrain.cpp:77-80)
            if (!s.condition_latents)
                throw InputError("condition mask lacks clean latents for its conditioned tokens");
            auto* m = static_cast<uint8_t*>(dalloc(static_cast<size_t>(N)));
            MGV_CUDA(cudaMemcpyAsync(m, s.conditioned, static_cast<size_t>(N), cudaMemcpyHostToDevice, stream_));
            d.cond = m;
            if (s.condition_latents != s.clean_rows) {
                // stage only the conditioned rows, one copy per contiguous run (a latent unit is a contiguous
                // run of rows in latent_rows order, dit.cpp:92-116); the other rows are never read
                auto* lat = static_cast<double*>(dalloc(sizeof(double) * N * D));
                for (int64_t i = 0; i < N;) {
                    if (!s.conditioned[i]) {
                        ++i;
                        continue;
                    }
                    int64_t j = i;
                    while (j < N && s.conditioned[j]) ++j;
                    MGV_CUDA(cudaMemcpyAsync(lat + i * D, s.condition_latents + i * D, sizeof(double) * (j - i) * D,
                                             cudaMemcpyHostToDevice, stream_));
                    i = j;
                }
                d.cond_lat = lat;
            }
        }
        ds[static_cast<size_t>(k)] = d;
    }
}

void Model::flow_step(int64_t n, const mgv_flow_sample* samples, const double* text, int64_t L, double fps,
                      double* loss, double* grad_norm, double* const* grads_out, double* const* v_out) {
    MGV_CUDA(cudaSetDevice(device_));
    if (n < 1) throw InputError("empty batch");
    if (L < 1 || L > 1 << 20) throw DimensionError("text embeddings must be (L, text_dim)");
    const int64_t D = cfg_.D();
    std::vector<DevSample> ds;
    std::vector<void*> allocs;
    auto dalloc = [&](size_t bytes) {
        void* p = nullptr;
        MGV_CUDA(cudaMallocAsync(&p, bytes, stream_));
        allocs.push_back(p);
        return p;
    };
    try {
        stage_samples(n, samples, ds, allocs);
        auto* tx = static_cast<double*>(dalloc(sizeof(double) * L * cfg_.text_dim));
        MGV_CUDA(cudaMemcpyAsync(tx, text, sizeof(double) * L * cfg_.text_dim, cudaMemcpyHostToDevice, stream_));
        std::vector<double*> vdev(n, nullptr);
        if (v_out)
            for (int64_t k = 0; k < n; ++k)
                if (v_out[k]) vdev[k] = static_cast<double*>(dalloc(sizeof(double) * ds[k].N * D));
        flow_step_dev(n, ds.data(), tx, L, fps, loss, grad_norm, v_out ? vdev.data() : nullptr);
        if (v_out)
            for (int64_t k = 0; k < n; ++k)
                if (v_out[k])
                    MGV_CUDA(cudaMemcpyAsync(v_out[k], vdev[k], sizeof(double) * ds[k].N * D, cudaMemcpyDeviceToHost,
                                             stream_));
        if (grads_out) download_grads(grads_out, dalloc);
        MGV_CUDA(cudaStreamSynchronize(stream_));
    } catch (...) {
        for (void* p : allocs) cudaFreeAsync(p, stream_);
        throw;
    }
    for (void* p : allocs) cudaFreeAsync(p, stream_);
}

template <class Alloc>
void Model::download_grads(double* const* grads_out, Alloc&& dalloc) {
    int64_t maxn = 0;
    for (auto* p : sorted_) maxn = std::max(maxn, p->numel_full);
    auto* gd = static_cast<double*>(dalloc(sizeof(double) * maxn));
    float* ga = tp_ > 1 ? static_cast<float*>(dalloc(sizeof(float) * maxn)) : nullptr;
    float* gb = tp_ > 1 ? static_cast<float*>(dalloc(sizeof(float) * maxn)) : nullptr;
    for (size_t k = 0; k < sorted_.size(); ++k) {
        if (!grads_out[k] && !(tp_ > 1 && !tp_virtual_ && sorted_[k]->shard)) continue;  // gathers are collective
        const DevParam& q = *sorted_[k];
        const float* gsrc = full_view(q, q.grad, ga, gb);
        if (!grads_out[k]) continue;
        f32_to_f64<<<grid_of(q.numel_full), 256, 0, stream_>>>(gsrc, q.numel_full, gd);
        ::mgv::note_launch();
        MGV_CUDA(cudaMemcpyAsync(grads_out[k], gd, sizeof(double) * q.numel_full, cudaMemcpyDeviceToHost, stream_));
        MGV_CUDA(cudaStreamSynchronize(stream_));
    }
}

void Model::eval_records(int64_t n, const mgv_eval_sample* recs, const double* weights, double* errs, double* loss,
                         double* grad_norm, double* const* grads_out) {
    MGV_CUDA(cudaSetDevice(device_));
    if (n < 1) throw InputError("empty batch");
    if (!recs || !errs || !loss) throw InputError("null argument");
    std::vector<mgv_flow_sample> fs(static_cast<size_t>(n));
    for (int64_t k = 0; k < n; ++k) {
        if (!recs[k].text || recs[k].L < 1 || recs[k].L > 1 << 20)
            throw DimensionError("text embeddings must be (L, text_dim)");
        fs[static_cast<size_t>(k)] = recs[k].s;
    }
    std::vector<DevSample> ds;
    std::vector<void*> allocs;
    auto dalloc = [&](size_t bytes) {
        void* p = nullptr;
        MGV_CUDA(cudaMallocAsync(&p, bytes, stream_));
        allocs.push_back(p);
        return p;
    };
    try {
        stage_samples(n, fs.data(), ds, allocs);
        std::vector<const double*> tdev(static_cast<size_t>(n));
        std::vector<int64_t> Ls(static_cast<size_t>(n));
        std::vector<double> fpss(static_cast<size_t>(n));
        for (int64_t k = 0; k < n; ++k) {  // one device copy per distinct host text
            int64_t same = -1;
            for (int64_t j = 0; j < k && same < 0; ++j)
                if (recs[j].text == recs[k].text && recs[j].L == recs[k].L) same = j;
            if (same >= 0) {
                tdev[static_cast<size_t>(k)] = tdev[static_cast<size_t>(same)];
            } else {
                auto* tx = static_cast<double*>(dalloc(sizeof(double) * recs[k].L * cfg_.text_dim));
                MGV_CUDA(cudaMemcpyAsync(tx, recs[k].text, sizeof(double) * recs[k].L * cfg_.text_dim,
                                         cudaMemcpyHostToDevice, stream_));
                tdev[static_cast<size_t>(k)] = tx;
            }
            Ls[static_cast<size_t>(k)] = recs[k].L;
            fpss[static_cast<size_t>(k)] = recs[k].fps;
        }
        StepExtra ex;
        ex.text_dev = tdev.data();
        ex.L = Ls.data();
        ex.fps = fpss.data();
        ex.backward = weights != nullptr;
        std::vector<double> ones;
        if (weights) {
            ex.weight = weights;
        } else {
            ones.assign(static_cast<size_t>(n), 1.0);
            ex.weight = ones.data();
        }
        ex.errs = errs;
        double gn = 0.0;
        flow_step_dev(n, ds.data(), tdev[0], Ls[0], fpss[0], loss, &gn, nullptr, &ex);
        if (grad_norm) *grad_norm = gn;
        if (weights && grads_out) download_grads(grads_out, dalloc);
        MGV_CUDA(cudaStreamSynchronize(stream_));
    } catch (...) {
        for (void* p : allocs) cudaFreeAsync(p, stream_);
        throw;
    }
    for (void* p : allocs) cudaFreeAsync(p, stream_);
}

// ------------------------------------------------------------------ value API (forward only)
template <class T>
void Model::value_forward(const double* in, int64_t N, const int32_t* coords, const int64_t dims[3],
                          const double* text, int64_t L, const double* tau, double fps, double* out, bool velocity) {
    if (!have_params_) throw InputError("no parameters uploaded");
    WS& w = *ws_;
    cudaStream_t s = stream_;
    const int64_t H = cfg_.H(), D = cfg_.D();
    if (N != dims[0] * dims[1] * dims[2]) throw DimensionError("token count does not match the grid");
    // unique timesteps -> modulation rows (dit.cpp:239-242 validates each)
    std::vector<double> uniq;
    std::vector<int32_t> mid(static_cast<size_t>(N));
    std::unordered_map<uint64_t, int> seen;
    for (int64_t i = 0; i < N; ++i) {
        if (!(tau[i] >= 0.0 && tau[i] <= 1.0)) throw InputError("timestep outside [0, 1]");
        uint64_t key;
        std::memcpy(&key, &tau[i], sizeof(key));
        if (tau[i] == 0.0) key = 0;  // +0 / -0
        auto it = seen.find(key);
        if (it == seen.end()) {
            it = seen.emplace(key, static_cast<int>(uniq.size())).first;
            uniq.push_back(tau[i]);
        }
        mid[static_cast<size_t>(i)] = it->second;
    }
    w.N = N;
    w.L = L;
    w.n_u = static_cast<int>(uniq.size());
    w.esz = bf16_ ? 2 : 4;
    w.grads = false;
    w.tp = tp_;
    w.tp_slots = tp_slots();
    w.recompute = recompute_ && w.grads;
    set_tpose(w, cfg_);
    {
        Sizer sz{true, 0, &arena_};
        layout_ws(w, sz, cfg_, false);
        arena_.reserve(sz.bytes);
        arena_.reset();
        Sizer real{false, 0, &arena_};
        layout_ws(w, real, cfg_, false);
    }
    const int64_t in_cols = velocity ? D : H;
    double* din = nullptr;
    MGV_CUDA(cudaMallocAsync(&din, sizeof(double) * std::max(N * in_cols, L * cfg_.text_dim), s));
    MGV_CUDA(cudaMemcpyAsync(w.coords, coords, sizeof(int32_t) * 3 * N, cudaMemcpyHostToDevice, s));
    MGV_CUDA(cudaMemcpyAsync(w.mod_id, mid.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice, s));
    MGV_CUDA(cudaMemcpyAsync(w.taus, uniq.data(), sizeof(double) * uniq.size(), cudaMemcpyHostToDevice, s));
    MGV_CUDA(cudaMemcpyAsync(din, text, sizeof(double) * L * cfg_.text_dim, cudaMemcpyHostToDevice, s));
    convert_rows<T>(din, L * cfg_.text_dim, tp<T>(w.text), s);
    MGV_CUDA(cudaMemcpyAsync(din, in, sizeof(double) * N * in_cols, cudaMemcpyHostToDevice, s));
    float* outf = nullptr;
    MGV_CUDA(cudaMallocAsync(&outf, sizeof(float) * N * std::max(H, D), s));
    DevSample dummy;
    if (velocity) {
        convert_rows<T>(din, N * D, tp<T>(w.rows), s);
        forward_sample<T>(dummy, w.rows, uniq.data(), w.n_u, nullptr, fps, false, true, nullptr);
        f32_to_f64<<<grid_of(N * D), 256, 0, s>>>(w.V, N * D, din); ::mgv::note_launch();
        MGV_CUDA(cudaMemcpyAsync(out, din, sizeof(double) * N * D, cudaMemcpyDeviceToHost, s));
    } else {
        // tokens enter the residual stream directly (dit.cpp:369)
        f64_to_f32_bf16<<<grid_of(N * H), 256, 0, s>>>(din, N * H, w.X[0], nullptr); ::mgv::note_launch();
        forward_sample<T>(dummy, nullptr, uniq.data(), w.n_u, nullptr, fps, false, false, outf);
        f32_to_f64<<<grid_of(N * H), 256, 0, s>>>(outf, N * H, din); ::mgv::note_launch();
        MGV_CUDA(cudaMemcpyAsync(out, din, sizeof(double) * N * H, cudaMemcpyDeviceToHost, s));
    }
    MGV_CUDA(cudaFreeAsync(outf, s));
    MGV_CUDA(cudaFreeAsync(din, s));
    MGV_CUDA(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ tape seam: velocity_rows_graph as one node
template <class T>
__global__ void to_f64_kernel(const T* src, int64_t n, double* dst) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        dst[e] = static_cast<double>(static_cast<float>(src[e]));
}

// unique timesteps -> modulation rows (dit.cpp:239-242 validates each); mid[i] = row of token i
static void dedup_taus(const double* tau, int64_t N, std::vector<double>& uniq, std::vector<int32_t>& mid) {
    uniq.clear();
    mid.assign(static_cast<size_t>(N), 0);
    std::unordered_map<uint64_t, int> seen;
    for (int64_t i = 0; i < N; ++i) {
        if (!(tau[i] >= 0.0 && tau[i] <= 1.0)) throw InputError("timestep outside [0, 1]");
        uint64_t key;
        std::memcpy(&key, &tau[i], sizeof(key));
        if (tau[i] == 0.0) key = 0;  // +0 / -0
        auto it = seen.find(key);
        if (it == seen.end()) {
            it = seen.emplace(key, static_cast<int>(uniq.size())).first;
            uniq.push_back(tau[i]);
        }
        mid[static_cast<size_t>(i)] = it->second;
    }
}

template <class T>
void Model::velocity_graph_impl(const double* rows, int64_t N, const int32_t* coords, const int64_t dims[3],
                                const double* text, int64_t L, const double* tau, double fps, double* V_out,
                                double* const* taps_out, const double* dV, double* const* grads_out) {
    if (!have_params_) throw InputError("no parameters uploaded");
    if (!rows || !coords || !dims || !text || !tau) throw InputError("null argument");
    if (N < 1 || N != dims[0] * dims[1] * dims[2]) throw DimensionError("token count does not match the grid");
    if (L < 1 || L > 1 << 20) throw DimensionError("text embeddings must be (L, text_dim)");
    if (world_ > 1 || tp_ > 1) throw ConfigError("the tape node runs on a single-device context");
    WS& w = *ws_;
    cudaStream_t s = stream_;
    const int64_t H = cfg_.H(), D = cfg_.D();
    std::vector<double> uniq;
    std::vector<int32_t> mid;
    dedup_taus(tau, N, uniq, mid);
    if (dV)  // the backward row kernels keep two modulation rows per 64-token chunk (kernels_elem.cu chunk_rows)
        for (int64_t r0 = 0; r0 < N; r0 += kRowsPerChunk) {
            int a = mid[static_cast<size_t>(r0)], b = a;
            for (int64_t i = r0; i < std::min<int64_t>(N, r0 + kRowsPerChunk); ++i) {
                const int u = mid[static_cast<size_t>(i)];
                if (u != a && u != b && b != a) throw InputError("the device backward takes at most two distinct "
                                                                 "timesteps per 64 consecutive tokens");
                if (u != a) b = u;
            }
        }
    w.N = N;
    w.L = L;
    w.n_u = static_cast<int>(uniq.size());
    w.esz = bf16_ ? 2 : 4;
    w.grads = true;  // keeps every block's residual stream (the taps) and the backward's activations
    w.tp = tp_;
    w.tp_slots = tp_slots();
    w.recompute = recompute_ && w.grads;
    set_tpose(w, cfg_);
    {
        Sizer sz{true, 0, &arena_};
        layout_ws(w, sz, cfg_, true);
        arena_.reserve(sz.bytes);
        arena_.reset();
        Sizer real{false, 0, &arena_};
        layout_ws(w, real, cfg_, true);
    }
    double* din = nullptr;
    MGV_CUDA(cudaMallocAsync(&din, sizeof(double) * std::max({N * H, N * D, L * cfg_.text_dim}), s));
    MGV_CUDA(cudaMemcpyAsync(w.coords, coords, sizeof(int32_t) * 3 * N, cudaMemcpyHostToDevice, s));
    MGV_CUDA(cudaMemcpyAsync(w.mod_id, mid.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice, s));
    MGV_CUDA(cudaMemcpyAsync(w.taus, uniq.data(), sizeof(double) * uniq.size(), cudaMemcpyHostToDevice, s));
    MGV_CUDA(cudaMemcpyAsync(din, text, sizeof(double) * L * cfg_.text_dim, cudaMemcpyHostToDevice, s));
    convert_rows<T>(din, L * cfg_.text_dim, tp<T>(w.text), s);
    MGV_CUDA(cudaMemcpyAsync(din, rows, sizeof(double) * N * D, cudaMemcpyHostToDevice, s));
    convert_rows<T>(din, N * D, tp<T>(w.rows), s);
    DevSample dummy;
    forward_sample<T>(dummy, w.rows, uniq.data(), w.n_u, nullptr, fps, true, true, nullptr);
    auto out_f32 = [&](const float* src, int64_t n, double* host) {
        f32_to_f64<<<grid_of(n), 256, 0, s>>>(src, n, din);
        note_launch();
        MGV_CUDA(cudaMemcpyAsync(host, din, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
        MGV_CUDA(cudaStreamSynchronize(s));
    };
    if (V_out) out_f32(w.V, N * D, V_out);
    if (taps_out) {  // dit.cpp:326-332 tap order
        for (int i = 0; i <= cfg_.depth; ++i)
            if (taps_out[i]) out_f32(w.X[i], N * H, taps_out[i]);  // patch embedding, then each block's output
        if (double* y = taps_out[cfg_.depth + 1]) {               // final normed projection (dit.cpp:315)
            to_f64_kernel<T><<<grid_of(N * H), 256, 0, s>>>(tp<T>(w.Y), N * H, din);
            note_launch();
            MGV_CUDA(cudaMemcpyAsync(y, din, sizeof(double) * N * H, cudaMemcpyDeviceToHost, s));
            MGV_CUDA(cudaStreamSynchronize(s));
        }
        if (taps_out[cfg_.depth + 2]) out_f32(w.V, N * D, taps_out[cfg_.depth + 2]);
    }
    if (dV) {
        MGV_CUDA(cudaMemsetAsync(grad_buf_, 0, sizeof(float) * grad_numel_, s));
        MGV_CUDA(cudaMemcpyAsync(din, dV, sizeof(double) * N * D, cudaMemcpyHostToDevice, s));
        convert_rows<T>(din, N * D, tp<T>(w.dV), s);
        dp_overlap_ = false;
        backward_sample<T>(w.dV);
        if (grads_out) {
            std::vector<void*> allocs;
            auto dalloc = [&](size_t bytes) {
                void* p = nullptr;
                MGV_CUDA(cudaMallocAsync(&p, bytes, s));
                allocs.push_back(p);
                return p;
            };
            download_grads(grads_out, dalloc);
            for (void* p : allocs) MGV_CUDA(cudaFreeAsync(p, s));
        }
    }
    MGV_CUDA(cudaFreeAsync(din, s));
    MGV_CUDA(cudaStreamSynchronize(s));
}

void Model::velocity_graph(const double* rows, int64_t N, const int32_t* coords, const int64_t dims[3],
                           const double* text, int64_t L, const double* tau, double fps, double* V_out,
                           double* const* taps_out, const double* dV, double* const* grads_out) {
    MGV_CUDA(cudaSetDevice(device_));
    if (bf16_)
        velocity_graph_impl<__nv_bfloat16>(rows, N, coords, dims, text, L, tau, fps, V_out, taps_out, dV, grads_out);
    else
        velocity_graph_impl<float>(rows, N, coords, dims, text, L, tau, fps, V_out, taps_out, dV, grads_out);
}

// ------------------------------------------------------------------ boundary helpers (dit.cpp:257-265, 336-359)
void Model::patchify(const double* grid, int64_t U, int64_t h, int64_t w_, int64_t C, double* tokens,
                     int32_t* coords) {
    MGV_CUDA(cudaSetDevice(device_));
    if (!have_params_) throw InputError("no parameters uploaded");
    if (!grid || !tokens || !coords) throw InputError("null argument");
    if (U < 1 || h < 1 || w_ < 1 || C < 1) throw DimensionError("latent grid must be (U, h, w, C)");
    if (h % 2 != 0 || w_ % 2 != 0) throw DimensionError("patchify needs even spatial dims");  // dit.cpp:95
    if (C != cfg_.c_z) throw DimensionError("latent channels do not match c_z " + std::to_string(cfg_.c_z));
    cudaStream_t s = stream_;
    const int64_t H = cfg_.H(), D = cfg_.D(), N = U * (h / 2) * (w_ / 2);
    double *dg = nullptr, *dr = nullptr, *dout = nullptr;
    float *r32 = nullptr, *o32 = nullptr;
    int32_t* dc = nullptr;
    MGV_CUDA(cudaMallocAsync(&dg, sizeof(double) * N * D, s));
    MGV_CUDA(cudaMallocAsync(&dr, sizeof(double) * N * D, s));
    MGV_CUDA(cudaMallocAsync(&dout, sizeof(double) * N * H, s));
    MGV_CUDA(cudaMallocAsync(&r32, sizeof(float) * N * D, s));
    MGV_CUDA(cudaMallocAsync(&o32, sizeof(float) * N * H, s));
    MGV_CUDA(cudaMallocAsync(&dc, sizeof(int32_t) * 3 * N, s));
    MGV_CUDA(cudaMemcpyAsync(dg, grid, sizeof(double) * N * D, cudaMemcpyHostToDevice, s));
    latent_rows_gather(dg, int(U), int(h), int(w_), int(C), dr, dc, s);
    f64_to_f32_bf16<<<grid_of(N * D), 256, 0, s>>>(dr, N * D, r32, nullptr);
    note_launch();
    gemm(false, Mat{r32, D, Major::K}, Mat{P("dit.patch.w").f32, D, Major::K}, int(N), int(H), int(D),
         EpiF32{o32, H, P("dit.patch.b").f32, 1.0f, 0, int(N), int(H)}, s);  // dit.cpp:343
    f32_to_f64<<<grid_of(N * H), 256, 0, s>>>(o32, N * H, dout);
    note_launch();
    MGV_CUDA(cudaMemcpyAsync(tokens, dout, sizeof(double) * N * H, cudaMemcpyDeviceToHost, s));
    MGV_CUDA(cudaMemcpyAsync(coords, dc, sizeof(int32_t) * 3 * N, cudaMemcpyDeviceToHost, s));
    for (void* q : {static_cast<void*>(dg), static_cast<void*>(dr), static_cast<void*>(dout), static_cast<void*>(r32),
                    static_cast<void*>(o32), static_cast<void*>(dc)})
        MGV_CUDA(cudaFreeAsync(q, s));
    MGV_CUDA(cudaStreamSynchronize(s));
}

void Model::unpatchify(const double* tokens, int64_t N, const int32_t* coords, const int64_t dims[3], double* grid) {
    MGV_CUDA(cudaSetDevice(device_));
    if (!have_params_) throw InputError("no parameters uploaded");
    if (!tokens || !coords || !dims || !grid) throw InputError("null argument");
    if (N < 1 || N != dims[0] * dims[1] * dims[2]) throw DimensionError("token coords do not match the grid dims");
    cudaStream_t s = stream_;
    const int64_t H = cfg_.H(), D = cfg_.D(), C = cfg_.c_z;
    double *dt = nullptr, *dr = nullptr, *dg = nullptr;
    float *t32 = nullptr, *r32 = nullptr;
    int32_t *dc = nullptr, *seen = nullptr, *st = nullptr;
    MGV_CUDA(cudaMallocAsync(&dt, sizeof(double) * N * H, s));
    MGV_CUDA(cudaMallocAsync(&dr, sizeof(double) * N * D, s));
    MGV_CUDA(cudaMallocAsync(&dg, sizeof(double) * N * D, s));
    MGV_CUDA(cudaMallocAsync(&t32, sizeof(float) * N * H, s));
    MGV_CUDA(cudaMallocAsync(&r32, sizeof(float) * N * D, s));
    MGV_CUDA(cudaMallocAsync(&dc, sizeof(int32_t) * 3 * N, s));
    MGV_CUDA(cudaMallocAsync(&seen, sizeof(int32_t) * N, s));
    MGV_CUDA(cudaMallocAsync(&st, sizeof(int32_t), s));
    MGV_CUDA(cudaMemcpyAsync(dt, tokens, sizeof(double) * N * H, cudaMemcpyHostToDevice, s));
    MGV_CUDA(cudaMemcpyAsync(dc, coords, sizeof(int32_t) * 3 * N, cudaMemcpyHostToDevice, s));
    f64_to_f32_bf16<<<grid_of(N * H), 256, 0, s>>>(dt, N * H, t32, nullptr);
    note_launch();
    gemm(false, Mat{t32, H, Major::K}, Mat{P("dit.out.w").f32, H, Major::K}, int(N), int(D), int(H),
         EpiF32{r32, D, P("dit.out.b").f32, 1.0f, 0, int(N), int(D)}, s);  // dit.cpp:355
    f32_to_f64<<<grid_of(N * D), 256, 0, s>>>(r32, N * D, dr);
    note_launch();
    MGV_CUDA(cudaMemsetAsync(dg, 0, sizeof(double) * N * D, s));
    rows_to_grid_scatter(dr, dc, int(N), int(dims[0]), int(dims[1]), int(dims[2]), int(C), dg, seen, st, s);
    int32_t status = 0;
    MGV_CUDA(cudaMemcpyAsync(&status, st, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    MGV_CUDA(cudaMemcpyAsync(grid, dg, sizeof(double) * N * D, cudaMemcpyDeviceToHost, s));
    for (void* q : {static_cast<void*>(dt), static_cast<void*>(dr), static_cast<void*>(dg), static_cast<void*>(t32),
                    static_cast<void*>(r32), static_cast<void*>(dc), static_cast<void*>(seen), static_cast<void*>(st)})
        MGV_CUDA(cudaFreeAsync(q, s));
    MGV_CUDA(cudaStreamSynchronize(s));
    if (status == 1) throw DimensionError("token coord outside the grid");  // dit.cpp:129-130
    if (status == 2) throw DimensionError("duplicate token coord");         // dit.cpp:132
}

void Model::global_embed_host(const double* tau, int64_t N, double fps, double* g, double* block_scales) {
    MGV_CUDA(cudaSetDevice(device_));
    if (!have_params_) throw InputError("no parameters uploaded");
    if (!tau || !g || N < 1) throw InputError("need one timestep per token");
    cudaStream_t s = stream_;
    const int64_t H = cfg_.H();
    // unique timesteps (dit.cpp:239-242 validates each); g rows depend only on their timestep
    std::vector<double> uniq;
    std::vector<int32_t> mid(static_cast<size_t>(N));
    std::unordered_map<uint64_t, int> seen;
    for (int64_t i = 0; i < N; ++i) {
        if (!(tau[i] >= 0.0 && tau[i] <= 1.0)) throw InputError("timestep outside [0, 1]");
        uint64_t key;
        std::memcpy(&key, &tau[i], sizeof(key));
        if (tau[i] == 0.0) key = 0;
        auto it = seen.find(key);
        if (it == seen.end()) {
            it = seen.emplace(key, static_cast<int>(uniq.size())).first;
            uniq.push_back(tau[i]);
        }
        mid[static_cast<size_t>(i)] = it->second;
    }
    const int n_u = static_cast<int>(uniq.size());
    double *dtau = nullptr, *phi = nullptr, *z_in = nullptr, *h_in = nullptr, *dgu = nullptr;
    MGV_CUDA(cudaMallocAsync(&dtau, sizeof(double) * n_u, s));
    MGV_CUDA(cudaMallocAsync(&phi, sizeof(double) * (n_u + 1) * 32, s));
    MGV_CUDA(cudaMallocAsync(&z_in, sizeof(double) * (n_u + 1) * H, s));
    MGV_CUDA(cudaMallocAsync(&h_in, sizeof(double) * (n_u + 1) * H, s));
    MGV_CUDA(cudaMallocAsync(&dgu, sizeof(double) * n_u * H, s));
    MGV_CUDA(cudaMemcpyAsync(dtau, uniq.data(), sizeof(double) * n_u, cudaMemcpyHostToDevice, s));
    ::mgv::global_embed(dtau, n_u, fps, P("dit.gmlp.in.w").f32, P("dit.gmlp.in.b").f32, P("dit.gmlp.out.w").f32,
                        P("dit.gmlp.out.b").f32, int(H), phi, z_in, h_in, dgu, s);
    std::vector<double> gu(static_cast<size_t>(n_u * H));
    MGV_CUDA(cudaMemcpyAsync(gu.data(), dgu, sizeof(double) * n_u * H, cudaMemcpyDeviceToHost, s));
    for (void* q : {static_cast<void*>(dtau), static_cast<void*>(phi), static_cast<void*>(z_in),
                    static_cast<void*>(h_in), static_cast<void*>(dgu)})
        MGV_CUDA(cudaFreeAsync(q, s));
    MGV_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < N; ++i)
        std::memcpy(g + i * H, gu.data() + static_cast<size_t>(mid[static_cast<size_t>(i)]) * H, sizeof(double) * H);
    if (block_scales) {  // the per-block gscale parameters (dit.cpp:263)
        for (int64_t i = 0; i < cfg_.depth; ++i) {
            for (size_t k = 0; k < sorted_.size(); ++k)
                if (sorted_[k]->name == blk(static_cast<int>(i), "gscale"))
                    download_param(static_cast<int64_t>(k), block_scales + i * H);
        }
    }
}

// ------------------------------------------------------------------ sampler (flowtrain.cpp:111-172)
// x += coef * v in fp64 (the reference's Euler state is fp64), then impose: conditioned rows <- latents
__global__ void euler_impose_kernel(double* x, const float* v, int64_t N, int64_t D, double coef,
                                    const uint8_t* cond, const double* cl) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N * D; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / D;
        if (cond && cond[i])
            x[e] = cl[e];  // impose (flowtrain.cpp:111-117)
        else if (v)
            x[e] += coef * static_cast<double>(v[e]);
    }
}

template <class T>
void Model::sample_impl(const double* x_start, int64_t N, const int32_t* coords, const int64_t dims[3],
                        const double* text, int64_t L, const uint8_t* cond, const double* cond_latents,
                        int64_t steps, int direction, double fps, double* out) {
    if (!have_params_) throw InputError("no parameters uploaded");
    if (steps < 1) throw InputError("steps must be >= 1");  // flowtrain.cpp:137, :160
    if (N != dims[0] * dims[1] * dims[2] || N < 1) throw DimensionError("rows do not match the token grid");
    if (L < 1) throw DimensionError("text embeddings must be (L, text_dim)");
    const int64_t D = cfg_.D();
    bool any = false;
    if (cond) {  // validate_mask (flowtrain.cpp:61-81)
        std::vector<int> unit(static_cast<size_t>(dims[0]), -1);
        for (int64_t i = 0; i < N; ++i) {
            const int u = coords[3 * i];
            if (u < 0 || u >= dims[0]) throw DimensionError("condition mask does not match the token grid");
            const int f = cond[i] ? 1 : 0;
            int& seen = unit[static_cast<size_t>(u)];
            if (seen == -1)
                seen = f;
            else if (seen != f)
                throw InputError("conditioned tokens must cover whole latent units");
            any = any || f;
        }
        if (any && !cond_latents) throw InputError("condition mask lacks clean latents for its conditioned tokens");
    }
    WS& w = *ws_;
    cudaStream_t s = stream_;
    w.N = N;
    w.L = L;
    w.n_u = any ? 2 : 1;  // per-token timesteps {tc, 0 at conditioned tokens} (flowtrain.cpp:119-124)
    w.esz = bf16_ ? 2 : 4;
    w.grads = false;
    w.tp = tp_;
    w.tp_slots = tp_slots();
    w.recompute = recompute_ && w.grads;
    set_tpose(w, cfg_);
    {
        Sizer sz{true, 0, &arena_};
        layout_ws(w, sz, cfg_, false);
        arena_.reserve(sz.bytes);
        arena_.reset();
        Sizer real{false, 0, &arena_};
        layout_ws(w, real, cfg_, false);
    }
    std::vector<int32_t> mid(static_cast<size_t>(N), 0);
    if (any)
        for (int64_t i = 0; i < N; ++i) mid[static_cast<size_t>(i)] = cond[i] ? 1 : 0;
    double *x = nullptr, *cl = nullptr, *din = nullptr;
    uint8_t* cm = nullptr;
    MGV_CUDA(cudaMallocAsync(&x, sizeof(double) * N * D, s));
    MGV_CUDA(cudaMallocAsync(&din, sizeof(double) * L * cfg_.text_dim, s));
    if (any) {
        MGV_CUDA(cudaMallocAsync(&cl, sizeof(double) * N * D, s));
        MGV_CUDA(cudaMallocAsync(&cm, N, s));
        MGV_CUDA(cudaMemcpyAsync(cl, cond_latents, sizeof(double) * N * D, cudaMemcpyHostToDevice, s));
        MGV_CUDA(cudaMemcpyAsync(cm, cond, N, cudaMemcpyHostToDevice, s));
    }
    MGV_CUDA(cudaMemcpyAsync(x, x_start, sizeof(double) * N * D, cudaMemcpyHostToDevice, s));
    MGV_CUDA(cudaMemcpyAsync(w.coords, coords, sizeof(int32_t) * 3 * N, cudaMemcpyHostToDevice, s));
    MGV_CUDA(cudaMemcpyAsync(w.mod_id, mid.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice, s));
    MGV_CUDA(cudaMemcpyAsync(din, text, sizeof(double) * L * cfg_.text_dim, cudaMemcpyHostToDevice, s));
    convert_rows<T>(din, L * cfg_.text_dim, tp<T>(w.text), s);
    const int grid = grid_of(N * D);
    euler_impose_kernel<<<grid, 256, 0, s>>>(x, nullptr, N, D, 0.0, cm, cl);  // impose(x) before the first step
    note_launch();
    const double dt = 1.0 / static_cast<double>(steps);
    DevSample dummy;
    for (int64_t k = 0; k < steps; ++k) {
        const double tc = direction < 0 ? 1.0 - static_cast<double>(k) * dt : static_cast<double>(k) * dt;
        set_taus(w.taus, tc, s);  // {tc, 0}
        convert_rows<T>(x, N * D, tp<T>(w.rows), s);
        forward_sample<T>(dummy, w.rows, nullptr, w.n_u, nullptr, fps, false, true, nullptr);  // velocity
        euler_impose_kernel<<<grid, 256, 0, s>>>(x, w.V, N, D, direction < 0 ? -dt : dt, cm, cl);
        note_launch();
    }
    MGV_CUDA(cudaMemcpyAsync(out, x, sizeof(double) * N * D, cudaMemcpyDeviceToHost, s));
    for (void* q : {static_cast<void*>(x), static_cast<void*>(din), static_cast<void*>(cl), static_cast<void*>(cm)})
        if (q) MGV_CUDA(cudaFreeAsync(q, s));
    MGV_CUDA(cudaStreamSynchronize(s));
}

void Model::sample_rows(const double* x_start, int64_t N, const int32_t* coords, const int64_t dims[3],
                        const double* text, int64_t L, const uint8_t* cond, const double* cond_latents, int64_t steps,
                        int direction, double fps, double* out) {
    MGV_CUDA(cudaSetDevice(device_));
    if (bf16_)
        sample_impl<__nv_bfloat16>(x_start, N, coords, dims, text, L, cond, cond_latents, steps, direction, fps, out);
    else
        sample_impl<float>(x_start, N, coords, dims, text, L, cond, cond_latents, steps, direction, fps, out);
}

void Model::predict_velocity(const double* rows, int64_t N, const int32_t* coords, const int64_t dims[3],
                             const double* text, int64_t L, const double* tau, double fps, double* out) {
    MGV_CUDA(cudaSetDevice(device_));
    if (bf16_)
        value_forward<__nv_bfloat16>(rows, N, coords, dims, text, L, tau, fps, out, true);
    else
        value_forward<float>(rows, N, coords, dims, text, L, tau, fps, out, true);
}
void Model::dit_forward(const double* tokens, int64_t N, const int32_t* coords, const int64_t dims[3],
                        const double* text, int64_t L, const double* tau, double fps, double* out) {
    MGV_CUDA(cudaSetDevice(device_));
    if (bf16_)
        value_forward<__nv_bfloat16>(tokens, N, coords, dims, text, L, tau, fps, out, false);
    else
        value_forward<float>(tokens, N, coords, dims, text, L, tau, fps, out, false);
}

}  // namespace mgv
