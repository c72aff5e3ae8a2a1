// Attention launchers.  Per head h: O_h = softmax(Q_h K_h^T) V_h with no
// implicit scale (Tape::mha, autodiff.cpp:755-793: callers fold any scaling
// into q) and no mask.  Operands are token-major with a row stride (ld) and
// head h at column offset h*hd, so the QKV projection output is consumed in
// place.  Backward is recompute-based (LSE saved) and deterministic: dQ and
// dK/dV come from separate passes, no float atomics.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace mgv {

struct AttnProblem {
    const void* q;
    int64_t q_ld;
    const void* k;
    int64_t k_ld;
    const void* v;
    int64_t v_ld;
    void* o;
    int64_t o_ld;
    float* lse;  // [heads][Nq]
    int Nq, Nk, heads, hd;
    // tensor-core path: V^T ([heads*hd][>= Nk], row h*hd+d holds v[:, h*hd+d]); null -> computed internally
    const void* vt = nullptr;
    int64_t vt_ld = 0;
    // per-head stride of lse (and of the backward's Dvec); 0 -> Nq.  The tensor-core backward
    // streams lse/D with bulk copies and wants it padded to a multiple of 64.
    int64_t lse_ld = 0;
    // block-diagonal self-attention over packed samples (varlen): for the 128-row tile t, its segment is rows
    // [seg[2t], seg[2t+1]); segments start on 256-row boundaries, so no query / key tile straddles two.  null: one
    // segment [0, N).  Every tile runs exactly the key / query steps it would run alone.
    const int* seg = nullptr;
};

__host__ __device__ inline int64_t lse_stride(const AttnProblem& p) { return p.lse_ld ? p.lse_ld : p.Nq; }

struct AttnBwdProblem {
    AttnProblem f;
    const void* dO;
    int64_t do_ld;
    float* Dvec;  // [heads][Nq] scratch: rowsum(dO * O)
    void* dq;
    int64_t dq_ld;
    void* dk;
    int64_t dk_ld;
    void* dv;
    int64_t dv_ld;
    float* dkv_part;  // [q_splits][heads][Nk][2*hd] scratch when q_splits > 1
    int q_splits;
    // tensor-core path: transposed Q, K, dO ([heads*hd][>= N] rows); provided by the caller's scratch
    void* qt = nullptr;
    int64_t qt_ld = 0;
    void* kt = nullptr;
    int64_t kt_ld = 0;
    void* dot = nullptr;
    int64_t dot_ld = 0;
};

// IEEE-fp32 math on T storage (T = float or bf16): the parity path
template <class T>
void attn_fwd_simt(const AttnProblem& p, cudaStream_t s);
template <class T>
void attn_bwd_simt(const AttnBwdProblem& p, cudaStream_t s);

// D[h][q] = rowsum(dO * O) (bf16 operands), shared by both backward paths
void attn_bwd_dvec(const AttnBwdProblem& p, cudaStream_t s);

// tcgen05 flash attention (bf16 operands, fp32 softmax / accumulate); hd in {64, 128, 144, ...} (hd % 16 == 0)
bool attn_tc_supported(int hd, int Nk);
void attn_fwd_tc(const AttnProblem& p, cudaStream_t s);
void attn_bwd_tc(const AttnBwdProblem& p, cudaStream_t s);

}  // namespace mgv
