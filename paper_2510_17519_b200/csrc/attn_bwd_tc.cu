// tcgen05 flash-attention backward for sm_100a, deterministic (no atomics):
// the gradient of Tape::mha (autodiff.cpp:795-843) in two passes.
//
//   dK/dV pass  CTA per (128-key tile, head), loops over 64-query tiles:
//                 S^T = K Q^T,  dP^T = V dO^T          (TMEM; Q^T/dO^T tiles read MN-major)
//                 P^T = exp(S^T - lse), dS^T = P^T (dP^T - D)   (thread = key row)
//                 dV += P^T dO, dK += dS^T Q           (ONE N=hd MMA per step: dO^T/Q^T read K-major)
//   dQ pass     CTA per (128-query tile, head), loops over 64-key tiles:
//                 S = Q K^T, dP = dO V^T               (double-buffered in TMEM)
//                 dS = P (dP - D)                      (thread = query row)
//                 dQ += dS K                           (K^T tile read K-major, N = hd)
// The transposed operands (Q^T, K^T, V^T, dO^T: [heads*hd][tokens]) are made
// once per step by a tiled transpose, so no MMA ever splits head_dim 144 into
// 128 + 16.  The MMA warp issues the next tile's S/dP products under the
// current tile's elementwise work.
#include <algorithm>
#include <cfloat>
#include <vector>

#include "attn.h"
#include "gemm.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace mgv {

// dK/dV pass variant: 0 = single-CTA kernel (default), 1 = 2-CTA cluster kernel.  The cluster kernel is
// correct (tests/test_attn_gpu.py runs both) but measured 2.5x slower at 57.6K tokens: its two per-step
// cross-SM handoffs (P^T out, dS^T back) put ~3600 clk of exchange latency on every step; kept selectable
// (mgv_dev_set_dkv_pair) as the starting point for a deeper-pipelined exchange.
static int g_dkv_pair = 0;
// 0 = v8 (default: V in TMEM, P^T in its own columns), 1 = v5 (K in TMEM, P^T / dS^T aliased)
static int g_dkv_variant = 0;
static int g_dkv_cw = 2;  // compute warps per TMEM lane group in the v8 dK/dV pass (2 or 4)
// dQ pass variant: 3 = v10 (default: 128-key steps, Q in TMEM, dO in shared memory, dS over dP), 2 = v9 (Q and dO
// in shared memory), 0 = v7 (64-key steps, Q and dO in TMEM, dP single-buffered), 1 = v8 (Q in shared memory, dP
// double-buffered)
static int g_dq_variant = 3;
static int g_dq_cw = 2;  // compute warps per TMEM lane group in the v9 dQ pass (2 or 4)
// timing experiments only (tools/): bit 0 = compute warps skip TMEM traffic and math, bit 1 = no Q^T/dO^T TMA
__device__ int g_attn_dbg = 0;

namespace {

constexpr float kLog2e = 1.4426950408889634f;

#ifdef MGV_ATTN_TRACE  // development timeline of one CTA (tools/trace_attn.py); not in the product build
__device__ unsigned long long g_attn_trace[8][64];
__device__ unsigned long long g_attn_trace2[8][64];
#define ATR(ev, j)                                                                              \
    do {                                                                                        \
        if (blockIdx.x == 7 && blockIdx.y == 0 && (j) < 64) g_attn_trace[ev][j] = clock64();   \
    } while (0)
#define ATR2(ev, j)                                                                                  \
    do {                                                                                             \
        if ((blockIdx.x >> 1) == 7 && blockIdx.y == 0 && (j) < 64) g_attn_trace2[ev][j] = clock64(); \
    } while (0)
#define ATR8(ev, j)                                                                             \
    do {                                                                                        \
        if (blockIdx.x == 7 && blockIdx.y == 0 && (j) < 64) g_attn_trace2[ev][j] = clock64();  \
    } while (0)
#define ATR9(ev, j)                                                                             \
    do {                                                                                        \
        if (blockIdx.x == 6 && blockIdx.y == 0 && (j) < 64) g_attn_trace2[ev][j] = clock64();  \
    } while (0)
#else
#define ATR9(ev, j) \
    do {            \
    } while (0)
#define ATR8(ev, j) \
    do {            \
    } while (0)
#define ATR2(ev, j) \
    do {            \
    } while (0)
#define ATR(ev, j) \
    do {           \
    } while (0)
#endif

template <int HD>
struct BT {
    static constexpr int NF = HD / 64;
    static constexpr int TAIL = HD % 64;
    static constexpr int ROW_TILE = NF * 16384 + (TAIL ? 4096 : 0);  // 128 tokens x HD, K-major over hd
    static constexpr int T_TILE = HD * 128;                          // HD rows x 64 tokens (transposed, SW128)
};

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int HD>
__device__ __forceinline__ void load_row_tile(uint8_t* dst, const CUtensorMap* m128, const CUtensorMap* m32,
                                              uint64_t* bar, int col0, int row0) {
    using T = BT<HD>;
#pragma unroll
    for (int c = 0; c < T::NF; ++c) tma_load_2d(dst + c * 16384, m128, bar, col0 + c * 64, row0);
    if (T::TAIL) tma_load_2d(dst + T::NF * 16384, m32, bar, col0 + T::NF * 64, row0);
}

// D[128 x 64] = A[128 x HD] . B^T where A is a 128-row tile K-major over hd and B^T is an
// HD x 64 transposed tile read MN-major (N = 64 tokens, K = hd rows).
template <int HD>
__device__ __forceinline__ void mma_rows_x_t(uint32_t d, uint32_t a, uint32_t bt) {
    using T = BT<HD>;
    constexpr uint32_t id = idesc_bf16_f32(128, 64, false, true);
    int kk = 0;
#pragma unroll
    for (int c = 0; c < T::NF; ++c)
#pragma unroll
        for (int k = 0; k < 4; ++k, ++kk)
            umma_f16_ss(d, smem_desc(a + c * 16384 + k * 32, 16, 1024, kSwizzle128),
                        smem_desc(bt + kk * 2048, 16, 1024, kSwizzle128), id, kk > 0);
    if (T::TAIL)
        umma_f16_ss(d, smem_desc(a + T::NF * 16384, 16, 256, kSwizzle32),
                    smem_desc(bt + kk * 2048, 16, 1024, kSwizzle128), id, 1);
}

// D[128 x HD] (+)= A[128 x 64] . B where A is a 128 x 64 K-major chunk (smem) and B is the HD x 64
// transposed tile read K-major (N = HD rows, K = 64 tokens): one N = HD MMA per 16-token step.
template <int HD>
__device__ __forceinline__ void mma_chunk_x_t(uint32_t d, uint32_t a, uint32_t bt, bool acc_first) {
    constexpr uint32_t id = idesc_bf16_f32(128, HD, false, false);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
        umma_f16_ss(d, smem_desc(a + ks * 32, 16, 1024, kSwizzle128), smem_desc(bt + ks * 32, 16, 1024, kSwizzle128),
                    id, (acc_first || ks > 0) ? 1u : 0u);
}

// D[128 x HD] (+)= A[128 x 64] . B with A read from TMEM (bf16 packed 2 per column, 32 columns)
// and B the HD x 64 transposed tile read K-major: one N = HD MMA per 16-token step (TS form).
template <int HD>
__device__ __forceinline__ void mma_tmem_x_t(uint32_t d, uint32_t a_tmem, uint32_t bt, bool acc_first) {
    constexpr uint32_t id = idesc_bf16_f32(128, HD, false, false);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
        umma_f16_ts(d, a_tmem + ks * 8, smem_desc(bt + ks * 32, 16, 1024, kSwizzle128), id,
                    (acc_first || ks > 0) ? 1u : 0u);
}

// As mma_tmem_x_t, with the 64-token A operand split over the compute warps of a lane group: warp w
// owns tokens [w W, w W + W) and keeps their bf16 pairs at columns [a_tmem + w W, a_tmem + w W + W/2).
template <int HD, int W>
__device__ __forceinline__ void mma_tmem_split_x_t(uint32_t d, uint32_t a_tmem, uint32_t bt, bool acc_first) {
    constexpr uint32_t id = idesc_bf16_f32(128, HD, false, false);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
        umma_f16_ts(d, a_tmem + (16 * ks / W) * W + (16 * ks % W) / 2, smem_desc(bt + ks * 32, 16, 1024, kSwizzle128),
                    id, (acc_first || ks > 0) ? 1u : 0u);
}
template <int N>
__device__ __forceinline__ void tmem_ldn(uint32_t taddr, float* r) {
    if constexpr (N == 16)
        tmem_ld16(taddr, reinterpret_cast<uint32_t*>(r));
    else
        tmem_ld32(taddr, reinterpret_cast<uint32_t*>(r));
}
template <int N>
__device__ __forceinline__ void tmem_stn(uint32_t taddr, const uint32_t* r) {
    if constexpr (N == 8)
        tmem_st8(taddr, r);
    else
        tmem_st16(taddr, r);
}
constexpr int kCWq = 2;  // compute warps per TMEM lane group in the dQ pass

// thread row -> 64 bf16 values of a 128 x 64 SW128 K-major chunk
__device__ __forceinline__ void st_row64(uint8_t* chunk, int row, const uint32_t* pk) {
    const uint32_t base = smem_u32(chunk) + row * 128;
#pragma unroll
    for (int u = 0; u < 8; ++u)
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(base + ((u ^ (row & 7)) << 4)), "r"(pk[4 * u]),
                     "r"(pk[4 * u + 1]), "r"(pk[4 * u + 2]), "r"(pk[4 * u + 3]));
}

template <int HD>
__device__ __forceinline__ void store_acc_row(uint32_t taddr, __nv_bfloat16* out, bool valid, int c0 = 0,
                                              int c1 = HD / 16) {
#pragma unroll 1
    for (int c = c0; c < c1; ++c) {
        uint32_t r[16];
        tmem_ld16(taddr + c * 16, r);
        tmem_wait_ld();
        if (valid) {
            uint32_t o[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = pack_bf16(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1]));
            uint4* dst = reinterpret_cast<uint4*>(out + c * 16);
            dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
            dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
        }
    }
}

template <int HD>
__device__ __forceinline__ void store_acc_row_f32(uint32_t taddr, float* out, bool valid) {
#pragma unroll 1
    for (int c = 0; c < HD / 16; ++c) {
        uint32_t r[16];
        tmem_ld16(taddr + c * 16, r);
        tmem_wait_ld();
        if (valid) {
            float4* dst = reinterpret_cast<float4*>(out + c * 16);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                dst[e] = make_float4(__uint_as_float(r[4 * e]), __uint_as_float(r[4 * e + 1]),
                                     __uint_as_float(r[4 * e + 2]), __uint_as_float(r[4 * e + 3]));
        }
    }
}

// dV | dK = sum over the query splits in split order (deterministic), to bf16
__global__ void reduce_dkv_parts(const float* part, int splits, int Nk, int64_t W, __nv_bfloat16* dv, int64_t dv_ld,
                                 __nv_bfloat16* dk, int64_t dk_ld) {
    const int64_t n = (int64_t)Nk * 2 * W;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        float acc = 0.0f;
        for (int z = 0; z < splits; ++z) acc += part[(int64_t)z * n + e];
        const int64_t row = e / (2 * W), c = e % (2 * W);
        if (c < W)
            dv[row * dv_ld + c] = __float2bfloat16_rn(acc);
        else
            dk[row * dk_ld + (c - W)] = __float2bfloat16_rn(acc);
    }
}

struct BwdMaps {
    CUtensorMap a128, a32, b128, b32;  // row tiles (dkv: K, V ; dq: Q, dO)
    CUtensorMap ta, tb;                // transposed tiles (dkv: Q^T, dO^T ; dq: K^T, V^T)
};

}  // namespace

template <int HD>
__device__ __forceinline__ void mma_tmem_rows_x_t(uint32_t d, uint32_t a_tmem, uint32_t bt) {
    constexpr uint32_t id = idesc_bf16_f32(128, 64, false, true);
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk)
        umma_f16_ts(d, a_tmem + kk * 8, smem_desc(bt + kk * 2048, 16, 1024, kSwizzle128), id, kk > 0 ? 1u : 0u);
}


// =====================================================================================  dK / dV
// K stays in TMEM (the A operand of S^T = K Q^T, a TS MMA); V is an SS operand of dP^T = V dO^T.
// P^T (bf16) is written over the first half of S^T and dS^T over the first half of dP^T; the MMA
// issue order  dV(i) -> S^T(i+1) -> dK(i) -> dP^T(i+1)  keeps every overwrite behind its reader and
// lets the softmax of step i+1 run under dK(i) and dP^T(i+1).
// TMEM: S^T|P^T [0,64)  dP^T|dS^T [64,128)  dV [128,128+HD)  dK [DK,DK+HD)  K (bf16 pairs) after.
// gridDim.z > 1 splits the query range (few key tiles, e.g. cross-attention over 64 text tokens):
// split z then writes fp32 partial dV | dK rows to part[z] (Nk x 2 heads*HD) for reduce_dkv_parts.
template <int HD>
__global__ void __launch_bounds__(384, 1) attn_bwd_dkv_tc_kernel(const __grid_constant__ BwdMaps tm, AttnBwdProblem p,
                                                                 float* part) {
    constexpr int BKV = 128, BQ = 64, NST = 5;
    using T = BT<HD>;
    constexpr int S_COL = 0, DP_COL = 64, DV_COL = 128, DK_COL = 128 + ((HD + 15) / 16) * 16;
    constexpr int KA_COL = DK_COL + ((HD + 15) / 16) * 16;
    static_assert(KA_COL + HD / 2 <= 512, "TMEM budget");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sV = smem;
    uint8_t* sQt = sV + T::ROW_TILE;        // [NST]
    uint8_t* sdOt = sQt + NST * T::T_TILE;  // [NST]
    float* sLse = reinterpret_cast<float*>(sdOt + NST * T::T_TILE);  // [NST][64]
    float* sD = sLse + NST * BQ;                                      // [NST][64]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sD + NST * BQ);
    uint64_t* v_full = bars;
    uint64_t* qd_full = bars + 1;         // [NST]
    uint64_t* qd_empty = bars + 1 + NST;  // [NST]
    uint64_t* s_full = bars + 1 + 2 * NST;
    uint64_t* dp_full = s_full + 1;
    uint64_t* p_full = s_full + 2;
    uint64_t* ds_full = s_full + 3;
    uint64_t* acc_done = s_full + 4;
    uint64_t* ka_ready = s_full + 5;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 6);

    const AttnProblem& f = p.f;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int h = blockIdx.y, k0 = blockIdx.x * BKV;
    const int nq_all = (f.Nq + BQ - 1) / BQ;
    const int i0 = static_cast<int>((int64_t)blockIdx.z * nq_all / gridDim.z);
    const int nq = static_cast<int>((int64_t)(blockIdx.z + 1) * nq_all / gridDim.z) - i0;  // this split's tiles
    const int col = h * HD;

    if (threadIdx.x == 0) {
        mbar_init(v_full, 1);
        for (int i = 0; i < NST; ++i) {
            mbar_init(&qd_full[i], 1);
            mbar_init(&qd_empty[i], 1);
        }
        mbar_init(s_full, 1);
        mbar_init(dp_full, 1);
        mbar_init(p_full, 8);
        mbar_init(ds_full, 8);
        mbar_init(acc_done, 1);
        mbar_init(ka_ready, 4);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (elect_one()) {
            mbar_arrive_expect_tx(v_full, T::ROW_TILE);
            load_row_tile<HD>(sV, &tm.b128, &tm.b32, v_full, col, k0);
            for (int i = 0; i < nq; ++i) {
                const int st = i % NST;
                if (i >= NST) mbar_wait(&qd_empty[st], ((i / NST) - 1) & 1);
                // Q^T / dO^T tiles + this tile's lse and D rows (lse/D padded per head to a multiple of 64)
                mbar_arrive_expect_tx(&qd_full[st], 2 * T::T_TILE + 2 * BQ * 4);
                const int qt = (i0 + i) * BQ;
                tma_load_2d(sQt + st * T::T_TILE, &tm.ta, &qd_full[st], qt, col);
                tma_load_2d(sdOt + st * T::T_TILE, &tm.tb, &qd_full[st], qt, col);
                bulk_load(sLse + st * BQ, f.lse + (int64_t)h * lse_stride(f) + qt, BQ * 4, &qd_full[st]);
                bulk_load(sD + st * BQ, p.Dvec + (int64_t)h * lse_stride(f) + qt, BQ * 4, &qd_full[st]);
            }
        }
    } else if (warp == 1) {
        const uint32_t aV = smem_u32(sV);
        auto issue_s = [&](int i) {
            mma_tmem_rows_x_t<HD>(tmem + S_COL, tmem + KA_COL, smem_u32(sQt + (i % NST) * T::T_TILE));
            umma_commit(s_full);
        };
        auto issue_dp = [&](int i) {
            mma_rows_x_t<HD>(tmem + DP_COL, aV, smem_u32(sdOt + (i % NST) * T::T_TILE));
            umma_commit(dp_full);
        };
        mbar_wait(ka_ready, 0);
        mbar_wait(v_full, 0);
        if (nq > 0) {
            mbar_wait(&qd_full[0], 0);
            tc_fence_after();
            if (elect_one()) {
                issue_s(0);
                issue_dp(0);
            }
            __syncwarp();
        }
        for (int i = 0; i < nq; ++i) {
            const int st = i % NST;
            mbar_wait(p_full, i & 1);
            tc_fence_after();
            if (elect_one()) mma_tmem_split_x_t<HD, 32>(tmem + DV_COL, tmem + S_COL, smem_u32(sdOt + st * T::T_TILE), i > 0);
            __syncwarp();
            if (i + 1 < nq) {  // S^T_{i+1} overwrites P^T_i: issued after dV_i, which reads it
                mbar_wait(&qd_full[(i + 1) % NST], ((i + 1) / NST) & 1);
                tc_fence_after();
                if (elect_one()) issue_s(i + 1);
                __syncwarp();
            }
            mbar_wait(ds_full, i & 1);
            tc_fence_after();
            if (elect_one()) {
                mma_tmem_split_x_t<HD, 32>(tmem + DK_COL, tmem + DP_COL, smem_u32(sQt + st * T::T_TILE), i > 0);
                umma_commit(&qd_empty[st]);
                if (i + 1 < nq) issue_dp(i + 1);  // overwrites dS^T_i: after dK_i
                if (i == nq - 1) umma_commit(acc_done);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        // two warps per TMEM lane group: warp hf handles query columns [32 hf, 32 hf + 32) of each tile
        const int g = warp & 3, hf = (warp - 4) >> 2, row = g * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(g * 32) << 16;
        const int kv = k0 + row;
        const bool kvv = kv < f.Nk;
        if (hf == 0) {
            row_to_tmem<HD>(tmem + lane_base + KA_COL,
                            static_cast<const __nv_bfloat16*>(f.k) + (int64_t)(kvv ? kv : 0) * f.k_ld + col, kvv);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(ka_ready);
        }
        constexpr int HQ = BQ / 2;
        for (int i = 0; i < nq; ++i) {
            const int st = i % NST;
            mbar_wait(&qd_full[st], (i / NST) & 1);  // lse / D rows of this tile have landed
            mbar_wait(s_full, i & 1);
            tc_fence_after();
            float s[HQ], dp[HQ];
            tmem_ld32(tmem + lane_base + S_COL + hf * HQ, reinterpret_cast<uint32_t*>(s));
            tmem_wait_ld();
            const float* lse2 = sLse + st * BQ + hf * HQ;
            const float* Dq = sD + st * BQ + hf * HQ;
            const int qb = (i0 + i) * BQ + hf * HQ;
            const bool full = qb + HQ <= f.Nq;
            uint32_t pk[HQ / 2];
#pragma unroll
            for (int c = 0; c < HQ; c += 2) {
                const bool v0 = full || qb + c < f.Nq, v1 = full || qb + c + 1 < f.Nq;
                s[c] = v0 ? ex2f((s[c] - lse2[c]) * kLog2e) : 0.0f;  // lse rows are natural-log
                s[c + 1] = v1 ? ex2f((s[c + 1] - lse2[c + 1]) * kLog2e) : 0.0f;
                pk[c / 2] = pack_bf16(s[c], s[c + 1]);
            }
            tmem_st16(tmem + lane_base + S_COL + hf * HQ, pk);  // P^T over this warp's own S^T columns
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(p_full);
            mbar_wait(dp_full, i & 1);
            tc_fence_after();
            tmem_ld32(tmem + lane_base + DP_COL + hf * HQ, reinterpret_cast<uint32_t*>(dp));
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < HQ; c += 2)
                pk[c / 2] = pack_bf16(s[c] * (dp[c] - Dq[c]), s[c + 1] * (dp[c + 1] - Dq[c + 1]));  // autodiff.cpp:820
            tmem_st16(tmem + lane_base + DP_COL + hf * HQ, pk);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(ds_full);
        }
        if (nq > 0) mbar_wait(acc_done, 0);
        tc_fence_after();
        const bool valid = kvv && nq > 0;
        if (part) {  // fp32 partial rows of this query split: [dV | dK]
            const int64_t W = (int64_t)f.heads * HD;
            float* prow = part + ((int64_t)blockIdx.z * f.Nk + (kvv ? kv : 0)) * 2 * W + (hf ? W : 0) + col;
            store_acc_row_f32<HD>(tmem + lane_base + (hf ? DK_COL : DV_COL), prow, kvv);
        } else if (hf == 0) {
            store_acc_row<HD>(tmem + lane_base + DV_COL,
                              static_cast<__nv_bfloat16*>(p.dv) + (int64_t)kv * p.dv_ld + col, valid);
        } else {
            store_acc_row<HD>(tmem + lane_base + DK_COL,
                              static_cast<__nv_bfloat16*>(p.dk) + (int64_t)kv * p.dk_ld + col, valid);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

// =====================================================================================  dK / dV (v8)
// The default dK/dV pass.  Against v5 above it moves V (not K) into TMEM and gives P^T its own columns:
//   S^T  = K Q^T     SS (K row tile in shared memory)         -> free-running: S^T(i+1) is issued as soon as
//                                                                the compute warps have loaded S^T(i)
//   dP^T = V dO^T    TS (V columns [0,128) in TMEM, the 16-column tail of head_dim 144 one SS k-step)
//   dV  += P^T dO    TS (P^T in its own 32 columns)
//   dK  += dS^T Q    TS (dS^T written over the consumed dP^T columns)
// so neither dependency loop (S^T -> softmax -> dV, dP^T -> dS -> dK -> dP^T) waits on the other product's
// overwrite, and the one shared-memory-operand product is the one whose loop has slack.  Staging only 128
// of V's 144 columns in TMEM is what makes the 512-column budget close:
//   S^T [0,64)  P^T [64,96)  dP^T|dS^T [96,160)  dV [160,160+HD)  dK [.., +HD)  V (bf16 pairs) [.., +64)
template <int HD, int CW>
__global__ void __launch_bounds__(128 + 128 * CW, 1) attn_bwd_dkv_v8_kernel(const __grid_constant__ BwdMaps tm,
                                                                           AttnBwdProblem p, float* part) {
    constexpr int BKV = 128, BQ = 64, NST = 5;
    static_assert(CW == 2 || CW == 4, "2 or 4 compute warps per TMEM lane group");
    using T = BT<HD>;
    constexpr int VA = HD >= 128 ? 128 : HD;  // V columns staged in TMEM
    constexpr int VT = HD - VA;               // tail columns read from shared memory
    static_assert(VT == 0 || VT == 16, "head_dim tail must be one 16-column k-step");
    constexpr int HDP = ((HD + 15) / 16) * 16;
    constexpr int S_COL = 0, P_COL = 64, DP_COL = 96, DV_COL = 160, DK_COL = DV_COL + HDP, VA_COL = DK_COL + HDP;
    static_assert(VA_COL + VA / 2 <= 512, "TMEM budget");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sK = smem;
    uint8_t* sVt = sK + T::ROW_TILE;                       // 128 x 16 SW32 tail of V (HD = 144)
    uint8_t* sQt = sVt + (VT ? 4096 : 0);                  // [NST]
    uint8_t* sdOt = sQt + NST * T::T_TILE;                 // [NST]
    float* sLse = reinterpret_cast<float*>(sdOt + NST * T::T_TILE);  // [NST][64]
    float* sD = sLse + NST * BQ;                                      // [NST][64]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sD + NST * BQ);
    uint64_t* k_full = bars;
    uint64_t* qd_full = bars + 1;         // [NST]
    uint64_t* qd_empty = bars + 1 + NST;  // [NST]
    uint64_t* s_full = bars + 1 + 2 * NST;
    uint64_t* s_empty = s_full + 1;
    uint64_t* p_full = s_full + 2;
    uint64_t* pv_done = s_full + 3;
    uint64_t* dp_full = s_full + 4;
    uint64_t* ds_full = s_full + 5;
    uint64_t* acc_done = s_full + 6;
    uint64_t* va_ready = s_full + 7;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 8);

    const AttnProblem& f = p.f;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int h = blockIdx.y, k0 = blockIdx.x * BKV;
    const int nq_all = (f.Nq + BQ - 1) / BQ;
    const int i0 = static_cast<int>((int64_t)blockIdx.z * nq_all / gridDim.z);
    const int nq = static_cast<int>((int64_t)(blockIdx.z + 1) * nq_all / gridDim.z) - i0;  // this split's tiles
    const int col = h * HD;

    if (threadIdx.x == 0) {
        mbar_init(k_full, 1);
        for (int i = 0; i < NST; ++i) {
            mbar_init(&qd_full[i], 1);
            mbar_init(&qd_empty[i], 1);
        }
        mbar_init(s_full, 1);
        mbar_init(s_empty, 4 * CW);
        mbar_init(p_full, 4 * CW);
        mbar_init(pv_done, 1);
        mbar_init(dp_full, 1);
        mbar_init(ds_full, 4 * CW);
        mbar_init(acc_done, 1);
        mbar_init(va_ready, 4);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (elect_one()) {
            mbar_arrive_expect_tx(k_full, T::ROW_TILE + (VT ? 4096 : 0));
            load_row_tile<HD>(sK, &tm.a128, &tm.a32, k_full, col, k0);
            if (VT) tma_load_2d(sVt, &tm.b32, k_full, col + VA, k0);
            for (int i = 0; i < nq; ++i) {
                const int st = i % NST;
                if (i >= NST) mbar_wait(&qd_empty[st], ((i / NST) - 1) & 1);
                if ((g_attn_dbg & 2) && i >= NST) {  // timing experiment: reuse the resident tiles, no TMA
                    mbar_arrive(&qd_full[st]);
                    continue;
                }
                mbar_arrive_expect_tx(&qd_full[st], 2 * T::T_TILE + 2 * BQ * 4);
                const int qt = (i0 + i) * BQ;
                tma_load_2d(sQt + st * T::T_TILE, &tm.ta, &qd_full[st], qt, col);
                tma_load_2d(sdOt + st * T::T_TILE, &tm.tb, &qd_full[st], qt, col);
                bulk_load(sLse + st * BQ, f.lse + (int64_t)h * lse_stride(f) + qt, BQ * 4, &qd_full[st]);
                bulk_load(sD + st * BQ, p.Dvec + (int64_t)h * lse_stride(f) + qt, BQ * 4, &qd_full[st]);
            }
        }
    } else if (warp == 1) {
        const uint32_t aK = smem_u32(sK);
        auto issue_s = [&](int i) {  // S^T(i) = K Q^T(i)
            if (elect_one()) {
                mma_rows_x_t<HD>(tmem + S_COL, aK, smem_u32(sQt + (i % NST) * T::T_TILE));
                umma_commit(s_full);
            }
            __syncwarp();
        };
        auto issue_dp = [&](int i) {  // dP^T(i) = V dO^T(i): VA/16 TS k-steps + the SS tail
            if (elect_one()) {
                constexpr uint32_t id = idesc_bf16_f32(128, 64, false, true);
                const uint32_t bt = smem_u32(sdOt + (i % NST) * T::T_TILE);
#pragma unroll
                for (int kk = 0; kk < VA / 16; ++kk)
                    umma_f16_ts(tmem + DP_COL, tmem + VA_COL + kk * 8, smem_desc(bt + kk * 2048, 16, 1024, kSwizzle128),
                                id, kk > 0 ? 1u : 0u);
                if (VT)
                    umma_f16_ss(tmem + DP_COL, smem_desc(smem_u32(sVt), 16, 256, kSwizzle32),
                                smem_desc(bt + (VA / 16) * 2048, 16, 1024, kSwizzle128), id, 1u);
                umma_commit(dp_full);
            }
            __syncwarp();
        };
        mbar_wait(va_ready, 0);
        mbar_wait(k_full, 0);
        if (nq > 0) {
            mbar_wait(&qd_full[0], 0);
            tc_fence_after();
            issue_s(0);
            issue_dp(0);
        }
        // per step i:  S^T(i+1) [S^T(i) loaded] -> dV(i) [P^T(i)] -> dK(i) [dS^T(i)] -> dP^T(i+1) [after dK(i)]
        for (int i = 0; i < nq; ++i) {
            const int st = i % NST;
            if (lane == 0) ATR8(0, i);
            if (i + 1 < nq) {
                mbar_wait(s_empty, i & 1);
                mbar_wait(&qd_full[(i + 1) % NST], ((i + 1) / NST) & 1);
                tc_fence_after();
                issue_s(i + 1);
            }
            if (lane == 0) ATR8(1, i);
            mbar_wait(p_full, i & 1);
            tc_fence_after();
            if (lane == 0) ATR8(2, i);
            if (elect_one()) {
                mma_tmem_x_t<HD>(tmem + DV_COL, tmem + P_COL, smem_u32(sdOt + st * T::T_TILE), i > 0);
                umma_commit(pv_done);
            }
            __syncwarp();
            if (lane == 0) ATR8(3, i);
            mbar_wait(ds_full, i & 1);
            tc_fence_after();
            if (lane == 0) ATR8(4, i);
            if (elect_one()) {
                mma_tmem_split_x_t<HD, BQ / CW>(tmem + DK_COL, tmem + DP_COL, smem_u32(sQt + st * T::T_TILE), i > 0);
                umma_commit(&qd_empty[st]);
                if (i == nq - 1) umma_commit(acc_done);
            }
            __syncwarp();
            if (lane == 0) ATR8(5, i);
            if (i + 1 < nq) issue_dp(i + 1);  // overwrites dS^T(i): behind dK(i) in the tensor pipe
            if (lane == 0) ATR8(6, i);
        }
    } else if (warp >= 4) {
        // CW warps per TMEM lane group: warp hf handles query columns [HQ hf, HQ hf + HQ) of each tile
        const int g = warp & 3, hf = (warp - 4) >> 2, row = g * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(g * 32) << 16;
        const int kv = k0 + row;
        const bool kvv = kv < f.Nk;
        if (hf == 0) {
            row_to_tmem<VA>(tmem + lane_base + VA_COL,
                            static_cast<const __nv_bfloat16*>(f.v) + (int64_t)(kvv ? kv : 0) * f.v_ld + col, kvv);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(va_ready);
        }
        constexpr int HQ = BQ / CW;
        for (int i = 0; i < nq; ++i) {
            const int st = i % NST;
            mbar_wait(&qd_full[st], (i / NST) & 1);  // lse / D rows of this tile have landed
            mbar_wait(s_full, i & 1);
            tc_fence_after();
            if (warp == 4 && lane == 0) ATR8(7, i);
            float s[HQ], dp[HQ];
            if (CW == 2 && (g_attn_dbg & 1)) {  // timing experiment: barriers only, no TMEM traffic or math
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(s_empty);
                if (i >= 1) mbar_wait(pv_done, (i - 1) & 1);
                if (lane == 0) mbar_arrive(p_full);
                mbar_wait(dp_full, i & 1);
                tc_fence_after();
                __syncwarp();
                if (lane == 0) mbar_arrive(ds_full);
                continue;
            }
            tmem_ldn<HQ>(tmem + lane_base + S_COL + hf * HQ, s);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(s_empty);  // the MMA warp may issue S^T(i+1) over it
            const float* lse2 = sLse + st * BQ + hf * HQ;
            const float* Dq = sD + st * BQ + hf * HQ;
            const int qb = (i0 + i) * BQ + hf * HQ;
            const bool full = qb + HQ <= f.Nq;
            uint32_t pk[HQ / 2];
#pragma unroll
            for (int c = 0; c < HQ; c += 2) {
                const bool v0 = full || qb + c < f.Nq, v1 = full || qb + c + 1 < f.Nq;
                s[c] = v0 ? ex2f((s[c] - lse2[c]) * kLog2e) : 0.0f;  // lse rows are natural-log
                s[c + 1] = v1 ? ex2f((s[c + 1] - lse2[c + 1]) * kLog2e) : 0.0f;
                pk[c / 2] = pack_bf16(s[c], s[c + 1]);
            }
            if (i >= 1) {
                mbar_wait(pv_done, (i - 1) & 1);  // dV(i-1) has read P^T(i-1)
                tc_fence_after();
            }
            tmem_stn<HQ / 2>(tmem + lane_base + P_COL + hf * (HQ / 2), pk);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(p_full);
            mbar_wait(dp_full, i & 1);
            tc_fence_after();
            tmem_ldn<HQ>(tmem + lane_base + DP_COL + hf * HQ, dp);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < HQ; c += 2)
                pk[c / 2] = pack_bf16(s[c] * (dp[c] - Dq[c]), s[c + 1] * (dp[c + 1] - Dq[c + 1]));  // autodiff.cpp:820
            tmem_stn<HQ / 2>(tmem + lane_base + DP_COL + hf * HQ, pk);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(ds_full);
        }
        if (nq > 0) mbar_wait(acc_done, 0);
        tc_fence_after();
        const bool valid = kvv && nq > 0;
        if (part) {  // fp32 partial rows of this query split: [dV | dK]
            if (hf < 2) {
                const int64_t W = (int64_t)f.heads * HD;
                float* prow = part + ((int64_t)blockIdx.z * f.Nk + (kvv ? kv : 0)) * 2 * W + (hf ? W : 0) + col;
                store_acc_row_f32<HD>(tmem + lane_base + (hf ? DK_COL : DV_COL), prow, kvv);
            }
        } else {  // warps [0, CW/2) store dV, the others dK, each a share of the 16-column chunks
            constexpr int NC = HD / 16, HALF = CW / 2;
            const bool is_v = hf < HALF;
            const int part_i = is_v ? hf : hf - HALF;
            __nv_bfloat16* out = is_v ? static_cast<__nv_bfloat16*>(p.dv) + (int64_t)kv * p.dv_ld + col
                                      : static_cast<__nv_bfloat16*>(p.dk) + (int64_t)kv * p.dk_ld + col;
            store_acc_row<HD>(tmem + lane_base + (is_v ? DV_COL : DK_COL), out, valid, part_i * NC / HALF,
                              (part_i + 1) * NC / HALF);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

// =====================================================================================  dK / dV (v9, cta_group::2)
// v8's schedule on a 2-CTA cluster that owns 256 keys (128 per CTA): every product is one M = 256 UMMA
// (tcgen05.mma.cta_group::2) issued by the leader CTA, so one issuing thread drives both SMs' tensor pipes.
// A single thread issues a tcgen05.mma every ~35-45 clk, about the execution time of a 128 x 64 x 16
// MMA, so with M = 128 the MMA warp of v8 is issue-bound (26 MMAs per 64-query step) and every barrier wait
// drains the pipe; with M = 256 the same 26 instructions cover twice the work.
// Operand split (the pair convention: A rows and D lanes per CTA, B rows split in half):
//   S^T  (M keys, N = 64 queries):  B = Q[32 r .. 32 r + 32, :)     per CTA, K-major row tile (QS tile)
//   dP^T (M keys, N = 64 queries):  B = dO[32 r .. 32 r + 32, :)    per CTA, K-major row tile (OS tile)
//   dV   (M keys, N = hd):          B = dO^T[72 r .. 72 r + 72, :)  per CTA, K-major SW128   (OH tile)
//   dK   (M keys, N = hd):          B = Q^T[72 r .. 72 r + 72, :)   per CTA, K-major SW128   (QH tile)
// TMEM per CTA as v8 (its 128 key lanes).  Leader barriers (waited by the MMA warp) count both CTAs'
// compute warps; the leader's commits are multicast to both CTAs.
template <int HD>
struct PairT {
    static constexpr int HH = HD / 2;          // head_dim rows per CTA in the K-major tiles
    static constexpr int NF = HD / 64, TAIL = HD % 64;
    static constexpr int S_TILE = NF * 4096 + (TAIL ? 1024 : 0);  // 32 token rows x HD: SW128 chunks + SW32 tail
    static constexpr int H_TILE = HH * 128;    // HH rows x 64 tokens (128 B rows, SW128)
    static constexpr int STAGE = 2 * S_TILE + 2 * H_TILE;
};

template <int HD>
__global__ void __launch_bounds__(384, 1) attn_bwd_dkv_v9_kernel(const __grid_constant__ BwdMaps tm,
                                                                 const __grid_constant__ BwdMaps tp2,
                                                                 AttnBwdProblem p) {
    constexpr int BKV = 128, BQ = 64, NST = 5;
    using T = BT<HD>;
    using PT = PairT<HD>;
    constexpr int VA = HD >= 128 ? 128 : HD;
    constexpr int VT = HD - VA;
    static_assert(VT == 0 || VT == 16, "head_dim tail must be one 16-column k-step");
    static_assert(PT::HH % 8 == 0, "half head_dim must be whole 8-row swizzle atoms");
    constexpr int HDP = ((HD + 15) / 16) * 16;
    constexpr int S_COL = 0, P_COL = 64, DP_COL = 96, DV_COL = 160, DK_COL = DV_COL + HDP, VA_COL = DK_COL + HDP;
    static_assert(VA_COL + VA / 2 <= 512, "TMEM budget");
    constexpr uint16_t kPair = 0x3;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sK = smem;
    uint8_t* sVt = sK + T::ROW_TILE;
    uint8_t* sStage = sVt + (VT ? 4096 : 0);  // [NST] x {QS, OS, QH, OH}
    float* sLse = reinterpret_cast<float*>(sStage + NST * PT::STAGE);  // [NST][64]
    float* sD = sLse + NST * BQ;                                        // [NST][64]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sD + NST * BQ);
    uint64_t* k_full = bars;                // leader: both CTAs' K / V tail
    uint64_t* qd_full = bars + 1;           // [NST] leader: both CTAs' operand tiles
    uint64_t* qd_empty = bars + 1 + NST;    // [NST] each CTA (multicast commit)
    uint64_t* ld_full = bars + 1 + 2 * NST; // [NST] each CTA: its lse / D rows
    uint64_t* s_full = bars + 1 + 3 * NST;  // each CTA (multicast)
    uint64_t* s_empty = s_full + 1;         // leader, 16 arrivals
    uint64_t* p_full = s_full + 2;          // leader, 16
    uint64_t* pv_done = s_full + 3;         // each CTA (multicast)
    uint64_t* dp_full = s_full + 4;         // each CTA (multicast)
    uint64_t* ds_full = s_full + 5;         // leader, 16
    uint64_t* acc_done = s_full + 6;        // each CTA (multicast)
    uint64_t* va_ready = s_full + 7;        // leader, 8
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 8);
    auto qs = [&](int st) { return sStage + st * PT::STAGE; };
    auto os = [&](int st) { return sStage + st * PT::STAGE + PT::S_TILE; };
    auto qh = [&](int st) { return sStage + st * PT::STAGE + 2 * PT::S_TILE; };
    auto oh = [&](int st) { return sStage + st * PT::STAGE + 2 * PT::S_TILE + PT::H_TILE; };

    const AttnProblem& f = p.f;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int rank = static_cast<int>(cluster_ctarank());
    const bool leader = rank == 0;
    const int h = blockIdx.y, k0 = (blockIdx.x >> 1) * 2 * BKV + rank * BKV;
    const int nq = (f.Nq + BQ - 1) / BQ;
    const int col = h * HD;

    if (threadIdx.x == 0) {
        mbar_init(k_full, 1);
        for (int i = 0; i < NST; ++i) {
            mbar_init(&qd_full[i], 1);
            mbar_init(&qd_empty[i], 1);
            mbar_init(&ld_full[i], 1);
        }
        mbar_init(s_full, 1);
        mbar_init(s_empty, 16);
        mbar_init(p_full, 16);
        mbar_init(pv_done, 1);
        mbar_init(dp_full, 1);
        mbar_init(ds_full, 16);
        mbar_init(acc_done, 1);
        mbar_init(va_ready, 8);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc_pair<512>(tmem_slot);
    tc_fence_before();
    cluster_sync();  // both CTAs' barriers initialised before any remote arrival / multicast
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (elect_one()) {
            const uint32_t kf = mapa(smem_u32(k_full), 0), qf = mapa(smem_u32(qd_full), 0);
            if (leader) mbar_arrive_expect_tx(k_full, 2 * (T::ROW_TILE + (VT ? 4096 : 0)));
#pragma unroll
            for (int c = 0; c < T::NF; ++c) tma_load_2d_pair(sK + c * 16384, &tm.a128, kf, col + c * 64, k0);
            if (T::TAIL) tma_load_2d_pair(sK + T::NF * 16384, &tm.a32, kf, col + T::NF * 64, k0);
            if (VT) tma_load_2d_pair(sVt, &tm.b32, kf, col + VA, k0);
            for (int i = 0; i < nq; ++i) {
                const int st = i % NST;
                if (i >= NST) mbar_wait(&qd_empty[st], ((i / NST) - 1) & 1);
                const int q0 = i * BQ;
                if (leader) mbar_arrive_expect_tx(&qd_full[st], 2 * PT::STAGE);
                // Q / dO rows: this CTA's 32 queries of the step (K-major over head_dim)
#pragma unroll
                for (int c = 0; c < PT::NF; ++c) {
                    tma_load_2d_pair(qs(st) + c * 4096, &tp2.a128, qf + st * 8, col + c * 64, q0 + 32 * rank);
                    tma_load_2d_pair(os(st) + c * 4096, &tp2.b128, qf + st * 8, col + c * 64, q0 + 32 * rank);
                }
                if (PT::TAIL) {
                    tma_load_2d_pair(qs(st) + PT::NF * 4096, &tp2.a32, qf + st * 8, col + PT::NF * 64, q0 + 32 * rank);
                    tma_load_2d_pair(os(st) + PT::NF * 4096, &tp2.b32, qf + st * 8, col + PT::NF * 64, q0 + 32 * rank);
                }
                // Q^T / dO^T: this CTA's head_dim rows of the step's 64 queries (K-major over queries)
                tma_load_2d_pair(qh(st), &tp2.ta, qf + st * 8, q0, col + PT::HH * rank);
                tma_load_2d_pair(oh(st), &tp2.tb, qf + st * 8, q0, col + PT::HH * rank);
                mbar_arrive_expect_tx(&ld_full[st], 2 * BQ * 4);
                bulk_load(sLse + st * BQ, f.lse + (int64_t)h * lse_stride(f) + q0, BQ * 4, &ld_full[st]);
                bulk_load(sD + st * BQ, p.Dvec + (int64_t)h * lse_stride(f) + q0, BQ * 4, &ld_full[st]);
            }
        }
    } else if (warp == 1) {
        if (leader) {
            constexpr uint32_t id64 = idesc_bf16_f32(256, 64, false, false), idhd = idesc_bf16_f32(256, HD, false, false);
            // k-step kk (head_dim 16 kk ..) of a K-major 32-row tile: SW128 chunk kk / 4, or the SW32 tail
            auto bdesc = [&](uint32_t b, int kk) {
                return kk < 4 * PT::NF ? smem_desc(b + (kk / 4) * 4096 + (kk % 4) * 32, 16, 1024, kSwizzle128)
                                       : smem_desc(b + PT::NF * 4096, 16, 256, kSwizzle32);
            };
            auto issue_s = [&](int i) {  // S^T(i) = K Q^T(i)
                if (elect_one()) {
                    const uint32_t a = smem_u32(sK), b = smem_u32(qs(i % NST));
                    int kk = 0;
#pragma unroll
                    for (int c = 0; c < T::NF; ++c)
#pragma unroll
                        for (int k4 = 0; k4 < 4; ++k4, ++kk)
                            umma_f16_ss_pair(tmem + S_COL, smem_desc(a + c * 16384 + k4 * 32, 16, 1024, kSwizzle128),
                                             bdesc(b, kk), id64, kk > 0);
                    if (T::TAIL)
                        umma_f16_ss_pair(tmem + S_COL, smem_desc(a + T::NF * 16384, 16, 256, kSwizzle32), bdesc(b, kk),
                                         id64, 1u);
                    umma_commit_pair_mc(s_full, kPair);
                }
                __syncwarp();
            };
            auto issue_dp = [&](int i) {  // dP^T(i) = V dO^T(i)
                if (elect_one()) {
                    const uint32_t b = smem_u32(os(i % NST));
#pragma unroll
                    for (int kk = 0; kk < VA / 16; ++kk)
                        umma_f16_ts_pair(tmem + DP_COL, tmem + VA_COL + kk * 8, bdesc(b, kk), id64, kk > 0 ? 1u : 0u);
                    if (VT)
                        umma_f16_ss_pair(tmem + DP_COL, smem_desc(smem_u32(sVt), 16, 256, kSwizzle32), bdesc(b, VA / 16),
                                         id64, 1u);
                    umma_commit_pair_mc(dp_full, kPair);
                }
                __syncwarp();
            };
            mbar_wait(va_ready, 0);
            mbar_wait(k_full, 0);
            if (nq > 0) {
                mbar_wait(&qd_full[0], 0);
                tc_fence_after();
                issue_s(0);
                issue_dp(0);
            }
            for (int i = 0; i < nq; ++i) {
                const int st = i % NST;
                if (lane == 0) ATR9(0, i);
                if (i + 1 < nq) {
                    mbar_wait(s_empty, i & 1);
                    mbar_wait(&qd_full[(i + 1) % NST], ((i + 1) / NST) & 1);
                    tc_fence_after();
                    issue_s(i + 1);
                }
                if (lane == 0) ATR9(1, i);
                mbar_wait(p_full, i & 1);
                tc_fence_after();
                if (lane == 0) ATR9(2, i);
                if (elect_one()) {  // dV += P^T dO
                    const uint32_t b = smem_u32(oh(st));
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks)
                        umma_f16_ts_pair(tmem + DV_COL, tmem + P_COL + ks * 8, smem_desc(b + ks * 32, 16, 1024, kSwizzle128),
                                         idhd, (i > 0 || ks > 0) ? 1u : 0u);
                    umma_commit_pair_mc(pv_done, kPair);
                }
                __syncwarp();
                if (lane == 0) ATR9(3, i);
                mbar_wait(ds_full, i & 1);
                tc_fence_after();
                if (lane == 0) ATR9(4, i);
                if (elect_one()) {  // dK += dS^T Q  (dS^T split over the two warps' query halves, as v8)
                    const uint32_t b = smem_u32(qh(st));
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks)
                        umma_f16_ts_pair(tmem + DK_COL, tmem + DP_COL + (16 * ks / 32) * 32 + (16 * ks % 32) / 2,
                                         smem_desc(b + ks * 32, 16, 1024, kSwizzle128), idhd, (i > 0 || ks > 0) ? 1u : 0u);
                    umma_commit_pair_mc(&qd_empty[st], kPair);
                    if (i == nq - 1) umma_commit_pair_mc(acc_done, kPair);
                }
                __syncwarp();
                if (lane == 0) ATR9(5, i);
                if (i + 1 < nq) issue_dp(i + 1);
                if (lane == 0) ATR9(6, i);
            }
        }
    } else if (warp >= 4) {
        const int g = warp & 3, hf = (warp - 4) >> 2, row = g * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(g * 32) << 16;
        const int kv = k0 + row;
        const bool kvv = kv < f.Nk;
        const uint32_t s_empty_l = mapa(smem_u32(s_empty), 0), p_full_l = mapa(smem_u32(p_full), 0);
        const uint32_t ds_full_l = mapa(smem_u32(ds_full), 0), va_ready_l = mapa(smem_u32(va_ready), 0);
        if (hf == 0) {
            row_to_tmem<VA>(tmem + lane_base + VA_COL,
                            static_cast<const __nv_bfloat16*>(f.v) + (int64_t)(kvv ? kv : 0) * f.v_ld + col, kvv);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(va_ready_l);
        }
        constexpr int HQ = BQ / 2;
        for (int i = 0; i < nq; ++i) {
            const int st = i % NST;
            mbar_wait(&ld_full[st], (i / NST) & 1);
            mbar_wait(s_full, i & 1);
            tc_fence_after();
            if (warp == 4 && lane == 0) ATR9(7, i);
            float s[HQ], dp[HQ];
            tmem_ld32(tmem + lane_base + S_COL + hf * HQ, reinterpret_cast<uint32_t*>(s));
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(s_empty_l);
            const float* lse2 = sLse + st * BQ + hf * HQ;
            const float* Dq = sD + st * BQ + hf * HQ;
            const int qb = i * BQ + hf * HQ;
            const bool full = qb + HQ <= f.Nq;
            uint32_t pk[HQ / 2];
#pragma unroll
            for (int c = 0; c < HQ; c += 2) {
                const bool v0 = full || qb + c < f.Nq, v1 = full || qb + c + 1 < f.Nq;
                s[c] = v0 ? ex2f((s[c] - lse2[c]) * kLog2e) : 0.0f;
                s[c + 1] = v1 ? ex2f((s[c + 1] - lse2[c + 1]) * kLog2e) : 0.0f;
                pk[c / 2] = pack_bf16(s[c], s[c + 1]);
            }
            if (i >= 1) {
                mbar_wait(pv_done, (i - 1) & 1);
                tc_fence_after();
            }
            tmem_st16(tmem + lane_base + P_COL + hf * (HQ / 2), pk);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(p_full_l);
            mbar_wait(dp_full, i & 1);
            tc_fence_after();
            tmem_ld32(tmem + lane_base + DP_COL + hf * HQ, reinterpret_cast<uint32_t*>(dp));
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < HQ; c += 2)
                pk[c / 2] = pack_bf16(s[c] * (dp[c] - Dq[c]), s[c + 1] * (dp[c + 1] - Dq[c + 1]));  // autodiff.cpp:820
            tmem_st16(tmem + lane_base + DP_COL + hf * HQ, pk);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(ds_full_l);
        }
        if (nq > 0) mbar_wait(acc_done, 0);
        tc_fence_after();
        const bool valid = kvv && nq > 0;
        if (hf == 0)
            store_acc_row<HD>(tmem + lane_base + DV_COL, static_cast<__nv_bfloat16*>(p.dv) + (int64_t)kv * p.dv_ld + col,
                              valid);
        else
            store_acc_row<HD>(tmem + lane_base + DK_COL, static_cast<__nv_bfloat16*>(p.dk) + (int64_t)kv * p.dk_ld + col,
                              valid);
    }
    tc_fence_before();
    cluster_sync();  // no CTA leaves while its peer may still arrive on / multicast into it
    tc_fence_after();
    if (warp == 2) tmem_dealloc_pair<512>(tmem);
}

// =====================================================================================  dK / dV, CTA pair
// The dK/dV pass with its TMEM split over a 2-CTA cluster that owns one 128-key tile: head_dim is cut
// into LO + HI columns (144 = 80 + 64, each a valid MMA N).  CTA 0 keeps K in TMEM and computes
// S^T = K Q^T and P = exp(S^T - lse); CTA 1 keeps V in TMEM and computes dP^T = V dO^T and
// dS = P (dP - D).  P^T and dS^T (bf16, 16 KB per step) are exchanged through distributed shared
// memory, so each CTA accumulates dV and dK for its own head_dim columns:
//   CTA 0:  dV[:, :LO] += P^T dO[:, :LO]  (TS, P^T in TMEM)    dK[:, :LO] += dS^T Q[:, :LO]  (SS, received)
//   CTA 1:  dV[:, LO:] += P^T dO[:, LO:]  (SS, received)       dK[:, LO:] += dS^T Q[:, LO:]  (TS)
// Every product now has a TMEM-resident or 64-token shared-memory A operand instead of re-reading the
// 128 x 144 K / V tile from shared memory each step, and the per-SM tensor work per step drops from
// 4 to ~2.4 k-step units.  The exchange buffers are double-buffered; receivers release them with
// cluster-scope mbarrier arrivals (tensor-core reads via multicast tcgen05.commit).
// TMEM (per CTA): S^T|P^T or dP^T|dS^T [0,64) [64,128)   dV part [128, 128+W)   dK part after   K or V.
template <int HD>
struct PairSplit {
    static constexpr int LO = ((HD / 2 + 15) / 16) * 16, HI = HD - LO;
    static_assert(HI > 0 && HI % 16 == 0, "head_dim split must give two multiple-of-16 halves");
};

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "LAB_WAITC:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra.uni DONEC;\n\t"
        "bra.uni LAB_WAITC;\n\t"
        "DONEC:\n\t}" ::"r"(addr),
        "r"(parity), "r"(1000000)
        : "memory");
}
// Exchanged P^T / dS^T tiles are two 128 x 32 K-major SW64 tiles (query columns [0,32) and [32,64)), so
// the 32 rows x 32 columns a compute warp produces are one contiguous 2 KB block: the warp stages it in
// its own shared memory and one lane bulk-copies it into the peer CTA (cp.async.bulk shared::cluster),
// completing on the peer's mbarrier.
__device__ __forceinline__ uint32_t sw64_off(int row, int chunk) {
    return row * 64 + ((chunk ^ ((row >> 1) & 3)) << 4);
}
__device__ __forceinline__ void st_row_sw64(uint32_t block, int row, const uint32_t* pk) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(block + sw64_off(row, u)), "r"(pk[4 * u]),
                     "r"(pk[4 * u + 1]), "r"(pk[4 * u + 2]), "r"(pk[4 * u + 3])
                     : "memory");
}
__device__ __forceinline__ void ld_row_sw64(uint32_t block, int row, float* v) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        uint32_t w[4];
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                     : "r"(block + sw64_off(row, u)));
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
            v[8 * u + 2 * e] = f.x;
            v[8 * u + 2 * e + 1] = f.y;
        }
    }
}
__device__ __forceinline__ void bulk_copy_to_peer(uint32_t dst_cluster, uint32_t src, uint32_t bytes,
                                                  uint32_t bar_cluster) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     dst_cluster),
                 "r"(src), "r"(bytes), "r"(bar_cluster)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// remote arrive that also announces `bytes` of complete_tx still to come on that barrier phase
__device__ __forceinline__ void mbar_arrive_expect_tx_cluster(uint32_t bar_cluster, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(bar_cluster),
                 "r"(bytes)
                 : "memory");
}
// D[128 x N] (+)= A[128 x 64] . B with A the exchanged pair of SW64 tiles and B read K-major (N rows)
template <int N>
__device__ __forceinline__ void mma_x64pair_x_t(uint32_t d, uint32_t a, uint32_t bt, bool acc_first) {
    constexpr uint32_t id = idesc_bf16_f32(128, N, false, false);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
        umma_f16_ss(d, smem_desc(a + (ks >> 1) * 8192 + (ks & 1) * 32, 16, 512, kSwizzle64),
                    smem_desc(bt + ks * 32, 16, 1024, kSwizzle128), id, (acc_first || ks > 0) ? 1u : 0u);
}

template <int HD>
__global__ void __launch_bounds__(384, 1) attn_bwd_dkv_pair_kernel(const __grid_constant__ BwdMaps tm, AttnBwdProblem p) {
    constexpr int BKV = 128, BQ = 64, HQ = 32, NST = 4;
    using T = BT<HD>;
    constexpr int LO = PairSplit<HD>::LO, HI = PairSplit<HD>::HI;
    // TMEM: S^T / dP^T [0,64) [64,128); own packed P^T / dS^T [128,160) [160,192); dV part, dK part; K / V
    constexpr int X_COL = 128, DV_COL = 192, A_COL = DV_COL + 2 * LO;
    static_assert(A_COL + HD / 2 <= 512, "TMEM budget");
    constexpr int XB = BKV * BQ * 2;  // one exchanged bf16 tile (16 KB)
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQt = smem;                    // [NST]
    uint8_t* sdOt = sQt + NST * T::T_TILE;  // [NST]
    uint8_t* xbuf = sdOt + NST * T::T_TILE;  // [2] received tiles: CTA 0 <- dS^T, CTA 1 <- P^T
    uint8_t* stg = xbuf + 2 * XB;            // [2][8 warps] 2 KB staging blocks of the outgoing tile
    float* sRow = reinterpret_cast<float*>(stg + 2 * XB);  // [NST][64]: lse (CTA 0) or D (CTA 1)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sRow + NST * BQ);
    uint64_t* qd_full = bars;             // [NST]
    uint64_t* qd_empty = bars + NST;      // [NST]
    uint64_t* s_full = bars + 2 * NST;    // [2] S^T (CTA 0) / dP^T (CTA 1) in TMEM
    uint64_t* s_empty = s_full + 2;       // [2] ... read by the compute warps
    uint64_t* x_full = s_full + 4;        // [2] own packed P^T / dS^T stored to TMEM
    uint64_t* x_done = s_full + 6;        // [2] ... consumed by this CTA's MMA
    uint64_t* recv = s_full + 8;          // [2] peer's tile landed in xbuf
    uint64_t* xfree = s_full + 10;        // [2] the peer may overwrite my outgoing buffer b
    uint64_t* acc_done = s_full + 12;
    uint64_t* a_ready = s_full + 13;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 14);

    const AttnProblem& f = p.f;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cluster_ctarank(), peer = rank ^ 1;
    const int h = blockIdx.y, k0 = (blockIdx.x >> 1) * BKV;
    const int nq = (f.Nq + BQ - 1) / BQ;
    const int col = h * HD;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(&qd_full[i], 1);
            mbar_init(&qd_empty[i], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&s_full[b], 1);
            mbar_init(&s_empty[b], 8);
            mbar_init(&x_full[b], 8);
            mbar_init(&x_done[b], 1);
            mbar_init(&recv[b], 8);
            // CTA 0's outgoing P^T buffer is freed by CTA 1's dV MMA (commit) and its 8 compute warps;
            // CTA 1's outgoing dS^T buffer by CTA 0's dK MMA
            mbar_init(&xfree[b], rank == 0 ? 9 : 1);
        }
        mbar_init(acc_done, 1);
        mbar_init(a_ready, 4);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    cluster_sync();  // barriers of both CTAs initialised before any remote arrival
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t xbuf_peer = mapa(smem_u32(xbuf), peer);
    const uint32_t recv_peer = mapa(smem_u32(recv), peer);
    const uint32_t xfree_peer = mapa(smem_u32(xfree), peer);

    if (warp == 0) {
        if (elect_one()) {
            const float* rowsrc = rank == 0 ? f.lse : p.Dvec;
            for (int i = 0; i < nq; ++i) {
                const int st = i % NST;
                if (i >= NST) mbar_wait(&qd_empty[st], ((i / NST) - 1) & 1);
                mbar_arrive_expect_tx(&qd_full[st], 2 * T::T_TILE + BQ * 4);
                tma_load_2d(sQt + st * T::T_TILE, &tm.ta, &qd_full[st], i * BQ, col);
                tma_load_2d(sdOt + st * T::T_TILE, &tm.tb, &qd_full[st], i * BQ, col);
                bulk_load(sRow + st * BQ, rowsrc + (int64_t)h * lse_stride(f) + i * BQ, BQ * 4, &qd_full[st]);
            }
        }
    } else if (warp == 1) {
        // CTA 0: S^T(i) = K Q^T ; CTA 1: dP^T(i) = V dO^T   (TS, A resident in TMEM), two steps ahead
        auto issue_s = [&](int i) {
            const int st = i % NST;
            mbar_wait(&qd_full[st], (i / NST) & 1);
            if (i >= 2) mbar_wait(&s_empty[i & 1], ((i - 2) >> 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                mma_tmem_rows_x_t<HD>(tmem + (i & 1) * 64, tmem + A_COL,
                                      smem_u32((rank == 0 ? sQt : sdOt) + st * T::T_TILE));
                umma_commit(&s_full[i & 1]);
            }
            __syncwarp();
        };
        auto qt_of = [&](int i) { return smem_u32(sQt + (i % NST) * T::T_TILE); };
        auto dot_of = [&](int i) { return smem_u32(sdOt + (i % NST) * T::T_TILE); };
        mbar_wait(a_ready, 0);
        if (nq > 0) issue_s(0);
        if (nq > 1) issue_s(1);
        if (rank == 0) {
            // per step i:  S^T(i+2) -> dV(i) [own P^T_i] -> dK(i-1) [dS^T_{i-1} from CTA 1, one step behind]
            auto issue_dk = [&](int j) {
                mbar_wait_cluster(&recv[j & 1], (j >> 1) & 1);
                tc_fence_after();
                if (elect_one()) {
                    mma_x64pair_x_t<LO>(tmem + DV_COL + LO, smem_u32(xbuf + (j & 1) * XB), qt_of(j), j > 0);
                    umma_commit_mc(&xfree[j & 1], 1u << peer);  // CTA 1 may refill xbuf[j & 1]
                    umma_commit(&qd_empty[j % NST]);
                    if (j == nq - 1) umma_commit(acc_done);
                }
                __syncwarp();
            };
            for (int i = 0; i < nq; ++i) {
                const int b = i & 1;
                if (i + 2 < nq) issue_s(i + 2);
                mbar_wait(&x_full[b], (i >> 1) & 1);
                tc_fence_after();
                if (elect_one()) {
                    mma_tmem_x_t<LO>(tmem + DV_COL, tmem + X_COL + b * 32, dot_of(i), i > 0);
                    umma_commit(&x_done[b]);
                }
                __syncwarp();
                if (i >= 1) issue_dk(i - 1);
            }
            if (nq > 0) issue_dk(nq - 1);
        } else {
            // per step i:  dP^T(i+2) -> dV(i) [P^T_i from CTA 0] -> dK(i) [own dS^T_i]
            for (int i = 0; i < nq; ++i) {
                const int b = i & 1;
                if (i + 2 < nq) issue_s(i + 2);
                mbar_wait_cluster(&recv[b], (i >> 1) & 1);
                tc_fence_after();
                if (elect_one()) {
                    mma_x64pair_x_t<HI>(tmem + DV_COL, smem_u32(xbuf + b * XB), dot_of(i) + LO * 128, i > 0);
                    umma_commit_mc(&xfree[b], 1u << peer);  // (with CTA 1's compute warps) CTA 0 may refill
                }
                __syncwarp();
                mbar_wait(&x_full[b], (i >> 1) & 1);
                tc_fence_after();
                if (elect_one()) {
                    mma_tmem_x_t<HI>(tmem + DV_COL + HI, tmem + X_COL + b * 32, qt_of(i) + LO * 128, i > 0);
                    umma_commit(&x_done[b]);
                    umma_commit(&qd_empty[i % NST]);
                    if (i == nq - 1) umma_commit(acc_done);
                }
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        // two warps per TMEM lane group: warp hf handles query columns [32 hf, 32 hf + 32) of each step
        const int g = warp & 3, hf = (warp - 4) >> 2, row = g * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(g * 32) << 16;
        const int kv = k0 + row;
        const bool kvv = kv < f.Nk;
        if (hf == 0) {  // stage K (CTA 0) or V (CTA 1) rows as the A operand
            const void* src = rank == 0 ? f.k : f.v;
            const int64_t ld = rank == 0 ? f.k_ld : f.v_ld;
            row_to_tmem<HD>(tmem + lane_base + A_COL,
                            static_cast<const __nv_bfloat16*>(src) + (int64_t)(kvv ? kv : 0) * ld + col, kvv);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(a_ready);
        }
        for (int i = 0; i < nq; ++i) {
            const int st = i % NST, b = i & 1;
            mbar_wait(&qd_full[st], (i / NST) & 1);  // lse / D rows of this tile
            mbar_wait(&s_full[b], (i >> 1) & 1);
            tc_fence_after();
            if (warp == 4 && lane == 0) ATR2(rank * 4 + 0, i);
            float x[HQ];
            tmem_ld32(tmem + lane_base + b * 64 + hf * HQ, reinterpret_cast<uint32_t*>(x));
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[b]);
            const float* rv = sRow + st * BQ + hf * HQ;
            const int qb = i * BQ + hf * HQ;
            uint32_t pk[HQ / 2];
            if (rank == 0) {  // P = exp(S^T - lse)
                if (qb + HQ <= f.Nq) {
#pragma unroll
                    for (int c = 0; c < HQ; ++c) x[c] = ex2f((x[c] - rv[c]) * kLog2e);
                } else {
#pragma unroll
                    for (int c = 0; c < HQ; ++c) x[c] = qb + c < f.Nq ? ex2f((x[c] - rv[c]) * kLog2e) : 0.0f;
                }
            } else {  // dS = P (dP - D), P from CTA 0
                mbar_wait_cluster(&recv[b], (i >> 1) & 1);
                float pv[HQ];
                ld_row_sw64(smem_u32(xbuf + b * XB) + hf * (XB / 2) + g * 2048, lane, pv);
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(xfree_peer + b * 8);  // done reading xbuf[b]
#pragma unroll
                for (int c = 0; c < HQ; ++c) x[c] = pv[c] * (x[c] - rv[c]);  // autodiff.cpp:820
            }
#pragma unroll
            for (int c = 0; c < HQ; c += 2) pk[c / 2] = pack_bf16(x[c], x[c + 1]);
            if (i >= 2) {
                mbar_wait(&x_done[b], ((i - 2) >> 1) & 1);  // own MMA done with step i-2's packed tile
                tc_fence_after();
            }
            tmem_st16(tmem + lane_base + X_COL + b * 32 + hf * (HQ / 2), pk);
            tmem_wait_st();
            if (warp == 4 && lane == 0) ATR2(rank * 4 + 1, i);
            // stage this warp's 32 x 32 block (SW64) and bulk-copy it into the peer's tile
            const uint32_t blk = smem_u32(stg) + (b * 8 + hf * 4 + g) * 2048;
            if (i >= 2) {
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // step i-2's copy read
                __syncwarp();
            }
            st_row_sw64(blk, lane, pk);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (i >= 2) mbar_wait_cluster(&xfree[b], ((i - 2) >> 1) & 1);  // peer done with step i-2's tile
            if (warp == 4 && lane == 0) ATR2(rank * 4 + 2, i);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&x_full[b]);
                mbar_arrive_expect_tx_cluster(recv_peer + b * 8, 2048);
                bulk_copy_to_peer(xbuf_peer + b * XB + hf * (XB / 2) + g * 2048, blk, 2048, recv_peer + b * 8);
            }
            if (warp == 4 && lane == 0) ATR2(rank * 4 + 3, i);
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // outgoing copies done
        if (nq > 0) mbar_wait(acc_done, 0);
        tc_fence_after();
        const bool valid = kvv && nq > 0;
        const int W = rank == 0 ? LO : HI, c0 = rank == 0 ? 0 : LO;
        __nv_bfloat16* out = hf == 0 ? static_cast<__nv_bfloat16*>(p.dv) + (int64_t)kv * p.dv_ld
                                     : static_cast<__nv_bfloat16*>(p.dk) + (int64_t)kv * p.dk_ld;
        store_acc_row<HD>(tmem + lane_base + (hf == 0 ? DV_COL : DV_COL + W), out + col + c0, valid, 0, W / 16);
    }
    tc_fence_before();
    cluster_sync();  // no CTA leaves while its peer may still write into it
    tc_fence_after();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

// =====================================================================================  dQ
// Q and dO stay in TMEM for the whole CTA (they are the A operands of S = Q K^T and dP = dO V^T), so
// every MMA of this pass is TS-form: only the 64-token K^T / V^T tiles are read from shared memory,
// and the products run at the tensor rate instead of the shared-memory operand rate of SS MMAs.
// TMEM: S[b] [64b, 64b+64)  dP [128,192)  dS [192,224)  dQ [224,224+HD)  Q, dO (bf16 pairs) after.
template <int HD>
__global__ void __launch_bounds__(128 + 128 * kCWq, 1) attn_bwd_dq_tc_kernel(const __grid_constant__ BwdMaps tm, AttnBwdProblem p) {
    constexpr int BMQ = 128, BKV = 64, NST = 6;
    using T = BT<HD>;
    constexpr int DP_COL = 128, DS_COL = 192, DQ_COL = 224;
    constexpr int QA_COL = DQ_COL + ((HD + 15) / 16) * 16, DOA_COL = QA_COL + HD / 2;
    static_assert(DOA_COL + HD / 2 <= 512, "TMEM budget");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sKt = smem;                   // [NST]
    uint8_t* sVt = sKt + NST * T::T_TILE;  // [NST]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sVt + NST * T::T_TILE);
    uint64_t* kv_full = bars;             // [NST]
    uint64_t* kv_empty = bars + NST;      // [NST]
    uint64_t* s_full = bars + 2 * NST;    // [2]
    uint64_t* s_empty = s_full + 2;       // [2]
    uint64_t* dp_full = s_full + 4;
    uint64_t* dp_empty = s_full + 5;
    uint64_t* ds_full = s_full + 6;
    uint64_t* dq_done = s_full + 7;
    uint64_t* acc_done = s_full + 8;
    uint64_t* qa_ready = s_full + 9;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 10);

    const AttnProblem& f = p.f;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int h = blockIdx.y, q0 = blockIdx.x * BMQ;
    const int nkv = (f.Nk + BKV - 1) / BKV;
    const int col = h * HD;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_empty[i], 4 * kCWq);
        }
        mbar_init(dp_full, 1);
        mbar_init(dp_empty, 4 * kCWq);
        mbar_init(ds_full, 4 * kCWq);
        mbar_init(dq_done, 1);
        mbar_init(acc_done, 1);
        mbar_init(qa_ready, 8);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (elect_one()) {
            for (int j = 0; j < nkv; ++j) {
                const int b = j % NST;
                if (j >= NST) mbar_wait(&kv_empty[b], ((j / NST) - 1) & 1);
                mbar_arrive_expect_tx(&kv_full[b], 2 * T::T_TILE);
                tma_load_2d(sKt + b * T::T_TILE, &tm.ta, &kv_full[b], j * BKV, col);
                tma_load_2d(sVt + b * T::T_TILE, &tm.tb, &kv_full[b], j * BKV, col);
            }
        }
    } else if (warp == 1) {
        auto issue_dq = [&](int j) {
            const int b = j % NST;
            mma_tmem_x_t<HD>(tmem + DQ_COL, tmem + DS_COL, smem_u32(sKt + b * T::T_TILE), j > 0);
            umma_commit(dq_done);
            umma_commit(&kv_empty[b]);
        };
        auto issue_s = [&](int j) {  // S_j into buffer j & 1
            const int b = j % NST;
            mbar_wait(&kv_full[b], (j / NST) & 1);
            if (j >= 2) mbar_wait(&s_empty[j & 1], ((j - 2) >> 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                mma_tmem_rows_x_t<HD>(tmem + (j & 1) * 64, tmem + QA_COL, smem_u32(sKt + b * T::T_TILE));
                umma_commit(&s_full[j & 1]);
            }
            __syncwarp();
        };
        auto issue_dp = [&](int j) {
            if (elect_one()) {
                mma_tmem_rows_x_t<HD>(tmem + DP_COL, tmem + DOA_COL, smem_u32(sVt + (j % NST) * T::T_TILE));
                umma_commit(dp_full);
            }
            __syncwarp();
        };
        // issue order per step j:  S(j+2) [S_j read] -> dP(j+1) [dP_j read] -> dQ(j) [dS_j ready]
        mbar_wait(qa_ready, 0);
        if (nkv > 0) issue_s(0);
        if (nkv > 1) issue_s(1);
        if (nkv > 0) issue_dp(0);
        for (int j = 0; j < nkv; ++j) {
            if (j + 2 < nkv) issue_s(j + 2);
            if (lane == 0) ATR(0, j);
            if (j + 1 < nkv) {
                mbar_wait(dp_empty, j & 1);
                tc_fence_after();
                if (lane == 0) ATR(1, j);
                issue_dp(j + 1);
            }
            mbar_wait(ds_full, j & 1);
            tc_fence_after();
            if (lane == 0) ATR(2, j);
            if (elect_one()) {
                issue_dq(j);
                if (j == nkv - 1) umma_commit(acc_done);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        // two warps per TMEM lane group: warp hf handles key columns [32 hf, 32 hf + 32) of each tile
        const int g = warp & 3, hf = (warp - 4) >> 2, row = g * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(g * 32) << 16;
        const int q = q0 + row;
        const bool qv = q < f.Nq;
        const int64_t qi = qv ? q : 0;
        if (hf < 2) {  // warp slices 0 / 1 stage Q / dO into TMEM
            if (hf == 0)
                row_to_tmem<HD>(tmem + lane_base + QA_COL, static_cast<const __nv_bfloat16*>(f.q) + qi * f.q_ld + col,
                                qv);
            else
                row_to_tmem<HD>(tmem + lane_base + DOA_COL,
                                static_cast<const __nv_bfloat16*>(p.dO) + qi * p.do_ld + col, qv);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(qa_ready);
        }
        const float lse2 = qv ? f.lse[(int64_t)h * lse_stride(f) + q] * kLog2e : 0.0f;
        const float Dq = qv ? p.Dvec[(int64_t)h * lse_stride(f) + q] : 0.0f;
        constexpr int HK = BKV / kCWq;
        // Software-pipelined like the dK/dV pass: iteration j loads S_{j+1} and dP_j together and computes
        // dS_j next to P_{j+1}.
        auto softmax = [&](float* x, int j) {  // x <- exp(x - lse) for key tile j (zero past Nk)
            const int kb = j * BKV + hf * HK;
            if (kb + HK <= f.Nk) {
#pragma unroll
                for (int c = 0; c < HK; ++c) x[c] = ex2f(fmaf(x[c], kLog2e, -lse2));
            } else {
#pragma unroll
                for (int c = 0; c < HK; ++c) x[c] = kb + c < f.Nk ? ex2f(fmaf(x[c], kLog2e, -lse2)) : 0.0f;
            }
        };
        float pr[HK];
        if (g_attn_dbg & 1) {  // timing experiment: barriers only, no TMEM traffic or math (wrong results)
            for (int j = 0; j < nkv; ++j) {
                if (j == 0) {
                    mbar_wait(&s_full[0], 0);
                    if (lane == 0) mbar_arrive(&s_empty[0]);
                }
                if (j + 1 < nkv) mbar_wait(&s_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
                mbar_wait(dp_full, j & 1);
                tc_fence_after();
                __syncwarp();
                if (lane == 0) {
                    if (j + 1 < nkv) mbar_arrive(&s_empty[(j + 1) & 1]);
                    mbar_arrive(dp_empty);
                }
                if (j >= 1) mbar_wait(dq_done, (j - 1) & 1);
                if (lane == 0) mbar_arrive(ds_full);
            }
        } else {
        if (nkv > 0) {
            mbar_wait(&s_full[0], 0);
            tc_fence_after();
            tmem_ldn<HK>(tmem + lane_base + hf * HK, pr);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[0]);
            softmax(pr, 0);
        }
        for (int j = 0; j < nkv; ++j) {
            const bool more = j + 1 < nkv;
            float sn[HK], dp[HK];
            if (more) {
                mbar_wait(&s_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
                tc_fence_after();
                tmem_ldn<HK>(tmem + lane_base + ((j + 1) & 1) * 64 + hf * HK, sn);
            }
            if (warp == 4 && lane == 0) ATR(3, j);
            mbar_wait(dp_full, j & 1);
            tc_fence_after();
            if (warp == 4 && lane == 0) ATR(4, j);
            tmem_ldn<HK>(tmem + lane_base + DP_COL + hf * HK, dp);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (more) mbar_arrive(&s_empty[(j + 1) & 1]);
                mbar_arrive(dp_empty);
            }
            uint32_t dk[HK / 2];
#pragma unroll
            for (int c = 0; c < HK; c += 2)
                dk[c / 2] = pack_bf16(pr[c] * (dp[c] - Dq), pr[c + 1] * (dp[c + 1] - Dq));  // autodiff.cpp:820
            if (more) softmax(sn, j + 1);
            if (warp == 4 && lane == 0) ATR(5, j);
            if (j >= 1) {
                mbar_wait(dq_done, (j - 1) & 1);  // dQ += dS_{j-1} K has read the dS columns
                tc_fence_after();
            }
            tmem_stn<HK / 2>(tmem + lane_base + DS_COL + hf * (HK / 2), dk);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(ds_full);
            if (warp == 4 && lane == 0) ATR(6, j);
#pragma unroll
            for (int c = 0; c < HK; ++c) pr[c] = sn[c];
        }
        }
        if (nkv > 0) mbar_wait(acc_done, 0);
        tc_fence_after();
        constexpr int NC = HD / 16;
        store_acc_row<HD>(tmem + lane_base + DQ_COL, static_cast<__nv_bfloat16*>(p.dq) + (int64_t)q * p.dq_ld + col,
                          qv && nkv > 0, hf * NC / kCWq, (hf + 1) * NC / kCWq);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

// =====================================================================================  dQ (v8)
// The dQ pass with dP double-buffered: Q moves from TMEM to a shared-memory row tile (S = Q K^T becomes an
// SS product), which frees the 64 TMEM columns of a second dP buffer.  Both products are then issued two
// key tiles ahead, so the dP round trip (MMA -> compute warps -> MMA) leaves the critical path.
// TMEM: S[b] [64b, 64b+64)  dP[b] [128+64b, ..)  dS [256,288)  dQ [288,288+HD)  dO (bf16 pairs) after.
template <int HD>
__global__ void __launch_bounds__(128 + 128 * kCWq, 1) attn_bwd_dq_v8_kernel(const __grid_constant__ BwdMaps tm,
                                                                            AttnBwdProblem p) {
    constexpr int BMQ = 128, BKV = 64, NST = 5;
    using T = BT<HD>;
    constexpr int DP_COL = 128, DS_COL = 256, DQ_COL = 288;
    constexpr int DOA_COL = DQ_COL + ((HD + 15) / 16) * 16;
    static_assert(DOA_COL + HD / 2 <= 512, "TMEM budget");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                            // 128 query rows x HD (K-major over hd)
    uint8_t* sKt = sQ + T::ROW_TILE;               // [NST]
    uint8_t* sVt = sKt + NST * T::T_TILE;          // [NST]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sVt + NST * T::T_TILE);
    uint64_t* kv_full = bars;             // [NST]
    uint64_t* kv_empty = bars + NST;      // [NST]
    uint64_t* s_full = bars + 2 * NST;    // [2]
    uint64_t* s_empty = s_full + 2;       // [2]
    uint64_t* dp_full = s_full + 4;       // [2]
    uint64_t* dp_empty = s_full + 6;      // [2]
    uint64_t* ds_full = s_full + 8;
    uint64_t* dq_done = s_full + 9;
    uint64_t* acc_done = s_full + 10;
    uint64_t* doa_ready = s_full + 11;
    uint64_t* q_full = s_full + 12;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 13);

    const AttnProblem& f = p.f;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int h = blockIdx.y, q0 = blockIdx.x * BMQ;
    const int nkv = (f.Nk + BKV - 1) / BKV;
    const int col = h * HD;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_empty[i], 4 * kCWq);
            mbar_init(&dp_full[i], 1);
            mbar_init(&dp_empty[i], 4 * kCWq);
        }
        mbar_init(ds_full, 4 * kCWq);
        mbar_init(dq_done, 1);
        mbar_init(acc_done, 1);
        mbar_init(doa_ready, 4);
        mbar_init(q_full, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (elect_one()) {
            mbar_arrive_expect_tx(q_full, T::ROW_TILE);
            load_row_tile<HD>(sQ, &tm.a128, &tm.a32, q_full, col, q0);
            for (int j = 0; j < nkv; ++j) {
                const int b = j % NST;
                if (j >= NST) mbar_wait(&kv_empty[b], ((j / NST) - 1) & 1);
                mbar_arrive_expect_tx(&kv_full[b], 2 * T::T_TILE);
                tma_load_2d(sKt + b * T::T_TILE, &tm.ta, &kv_full[b], j * BKV, col);
                tma_load_2d(sVt + b * T::T_TILE, &tm.tb, &kv_full[b], j * BKV, col);
            }
        }
    } else if (warp == 1) {
        const uint32_t aQ = smem_u32(sQ);
        auto issue_s = [&](int j) {  // S_j = Q K_j^T into buffer j & 1 (SS)
            const int b = j % NST;
            mbar_wait(&kv_full[b], (j / NST) & 1);
            if (j >= 2) mbar_wait(&s_empty[j & 1], ((j - 2) >> 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                mma_rows_x_t<HD>(tmem + (j & 1) * 64, aQ, smem_u32(sKt + b * T::T_TILE));
                umma_commit(&s_full[j & 1]);
            }
            __syncwarp();
        };
        auto issue_dp = [&](int j) {  // dP_j = dO V_j^T into buffer j & 1 (TS)
            if (j >= 2) mbar_wait(&dp_empty[j & 1], ((j - 2) >> 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                mma_tmem_rows_x_t<HD>(tmem + DP_COL + (j & 1) * 64, tmem + DOA_COL,
                                      smem_u32(sVt + (j % NST) * T::T_TILE));
                umma_commit(&dp_full[j & 1]);
            }
            __syncwarp();
        };
        // issue order per step j:  S(j+2) [S_j read] -> dP(j+2) [dP_j read] -> dQ(j) [dS_j ready]
        mbar_wait(doa_ready, 0);
        mbar_wait(q_full, 0);
        for (int j = 0; j < 2 && j < nkv; ++j) {
            issue_s(j);
            issue_dp(j);
        }
        for (int j = 0; j < nkv; ++j) {
            if (j + 2 < nkv) {
                issue_s(j + 2);
                issue_dp(j + 2);
            }
            mbar_wait(ds_full, j & 1);
            tc_fence_after();
            if (elect_one()) {
                const int b = j % NST;
                mma_tmem_x_t<HD>(tmem + DQ_COL, tmem + DS_COL, smem_u32(sKt + b * T::T_TILE), j > 0);
                umma_commit(dq_done);
                umma_commit(&kv_empty[b]);
                if (j == nkv - 1) umma_commit(acc_done);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        const int g = warp & 3, hf = (warp - 4) >> 2, row = g * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(g * 32) << 16;
        const int q = q0 + row;
        const bool qv = q < f.Nq;
        const int64_t qi = qv ? q : 0;
        if (hf == 0) {  // stage dO rows into TMEM (A operand of dP)
            row_to_tmem<HD>(tmem + lane_base + DOA_COL, static_cast<const __nv_bfloat16*>(p.dO) + qi * p.do_ld + col,
                            qv);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(doa_ready);
        }
        const float lse2 = qv ? f.lse[(int64_t)h * lse_stride(f) + q] * kLog2e : 0.0f;
        const float Dq = qv ? p.Dvec[(int64_t)h * lse_stride(f) + q] : 0.0f;
        constexpr int HK = BKV / kCWq;
        auto softmax = [&](float* x, int j) {
            const int kb = j * BKV + hf * HK;
            if (kb + HK <= f.Nk) {
#pragma unroll
                for (int c = 0; c < HK; ++c) x[c] = ex2f(fmaf(x[c], kLog2e, -lse2));
            } else {
#pragma unroll
                for (int c = 0; c < HK; ++c) x[c] = kb + c < f.Nk ? ex2f(fmaf(x[c], kLog2e, -lse2)) : 0.0f;
            }
        };
        float pr[HK];
        if (nkv > 0) {
            mbar_wait(&s_full[0], 0);
            tc_fence_after();
            tmem_ldn<HK>(tmem + lane_base + hf * HK, pr);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[0]);
            softmax(pr, 0);
        }
        for (int j = 0; j < nkv; ++j) {
            const bool more = j + 1 < nkv;
            float sn[HK], dp[HK];
            if (more) {
                mbar_wait(&s_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
                tc_fence_after();
                tmem_ldn<HK>(tmem + lane_base + ((j + 1) & 1) * 64 + hf * HK, sn);
            }
            mbar_wait(&dp_full[j & 1], (j >> 1) & 1);
            tc_fence_after();
            tmem_ldn<HK>(tmem + lane_base + DP_COL + (j & 1) * 64 + hf * HK, dp);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (more) mbar_arrive(&s_empty[(j + 1) & 1]);
                mbar_arrive(&dp_empty[j & 1]);
            }
            uint32_t dk[HK / 2];
#pragma unroll
            for (int c = 0; c < HK; c += 2)
                dk[c / 2] = pack_bf16(pr[c] * (dp[c] - Dq), pr[c + 1] * (dp[c + 1] - Dq));  // autodiff.cpp:820
            if (more) softmax(sn, j + 1);
            if (j >= 1) {
                mbar_wait(dq_done, (j - 1) & 1);  // dQ += dS_{j-1} K has read the dS columns
                tc_fence_after();
            }
            tmem_stn<HK / 2>(tmem + lane_base + DS_COL + hf * (HK / 2), dk);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(ds_full);
#pragma unroll
            for (int c = 0; c < HK; ++c) pr[c] = sn[c];
        }
        if (nkv > 0) mbar_wait(acc_done, 0);
        tc_fence_after();
        constexpr int NC = HD / 16;
        store_acc_row<HD>(tmem + lane_base + DQ_COL, static_cast<__nv_bfloat16*>(p.dq) + (int64_t)q * p.dq_ld + col,
                          qv && nkv > 0, hf * NC / kCWq, (hf + 1) * NC / kCWq);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

// =====================================================================================  dQ (v9)
// 128-key steps: every product is an N = 128 (S, dP) or K = 128 (dQ) MMA, so a step of the same work issues
// 26 instead of 44 tcgen05.mma instructions (one thread issues one per ~40 clk, which bounds v7).  To fit
// TMEM (S 128 + dP 128 + dS 64 + dQ 144 = 464 columns) Q and dO are shared-memory A operands (SS).
// K^T (S and dQ) and V^T (dP) have separate two-stage rings; the issue order S(j+1) -> dQ(j) -> dP(j+1)
// releases K^T(j) one product earlier than v7's order.
// TMEM: S [0,128)  dP [128,256)  dS [256,320)  dQ [320,320+HD).
template <int HD, int CW>
__global__ void __launch_bounds__(128 + 128 * CW, 1) attn_bwd_dq_v9_kernel(const __grid_constant__ BwdMaps tm,
                                                                          AttnBwdProblem p) {
    constexpr int BMQ = 128, BKV = 128, KW = BKV / CW;  // CW compute warps per TMEM lane group, KW keys each
    static_assert(KW == 32 || KW == 64, "32 or 64 keys per compute warp");
    using T = BT<HD>;
    constexpr int S_COL = 0, DP_COL = 128, DS_COL = 256, DQ_COL = 320;
    static_assert(DQ_COL + ((HD + 15) / 16) * 16 <= 512, "TMEM budget");
    constexpr int KV_STAGE = 2 * T::T_TILE;  // two 64-key transposed tiles
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sdO = sQ + T::ROW_TILE;
    uint8_t* sKt = sdO + T::ROW_TILE;  // [2]
    uint8_t* sVt = sKt + 2 * KV_STAGE;  // [2]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sVt + 2 * KV_STAGE);
    uint64_t* q_full = bars;
    uint64_t* kf = bars + 1;  // [2]
    uint64_t* ke = bars + 3;  // [2]
    uint64_t* vf = bars + 5;  // [2]
    uint64_t* ve = bars + 7;  // [2]
    uint64_t* s_full = bars + 9;
    uint64_t* s_empty = bars + 10;
    uint64_t* dp_full = bars + 11;
    uint64_t* dp_empty = bars + 12;
    uint64_t* ds_full = bars + 13;
    uint64_t* dq_done = bars + 14;
    uint64_t* acc_done = bars + 15;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

    const AttnProblem& f = p.f;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int h = blockIdx.y, q0 = blockIdx.x * BMQ;
    const int nkv = (f.Nk + BKV - 1) / BKV;
    const int col = h * HD;

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&kf[i], 1);
            mbar_init(&ke[i], 1);
            mbar_init(&vf[i], 1);
            mbar_init(&ve[i], 1);
        }
        mbar_init(s_full, 1);
        mbar_init(s_empty, 4 * CW);
        mbar_init(dp_full, 1);
        mbar_init(dp_empty, 4 * CW);
        mbar_init(ds_full, 4 * CW);
        mbar_init(dq_done, 1);
        mbar_init(acc_done, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (elect_one()) {
            mbar_arrive_expect_tx(q_full, 2 * T::ROW_TILE);
            load_row_tile<HD>(sQ, &tm.a128, &tm.a32, q_full, col, q0);
            load_row_tile<HD>(sdO, &tm.b128, &tm.b32, q_full, col, q0);
            for (int j = 0; j < nkv; ++j) {
                const int b = j & 1;
                if (j >= 2) mbar_wait(&ke[b], ((j >> 1) - 1) & 1);
                mbar_arrive_expect_tx(&kf[b], KV_STAGE);
                tma_load_2d(sKt + b * KV_STAGE, &tm.ta, &kf[b], j * BKV, col);
                tma_load_2d(sKt + b * KV_STAGE + T::T_TILE, &tm.ta, &kf[b], j * BKV + 64, col);
                if (j >= 2) mbar_wait(&ve[b], ((j >> 1) - 1) & 1);
                mbar_arrive_expect_tx(&vf[b], KV_STAGE);
                tma_load_2d(sVt + b * KV_STAGE, &tm.tb, &vf[b], j * BKV, col);
                tma_load_2d(sVt + b * KV_STAGE + T::T_TILE, &tm.tb, &vf[b], j * BKV + 64, col);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t id128 = idesc_bf16_f32(128, 128, false, true), idhd = idesc_bf16_f32(128, HD, false, false);
        // D[128 x 128] = A[128 x HD] (smem rows) . B^T with B^T the two-tile HD x 128 transposed stage (MN-major)
        auto rows_x_t2 = [&](uint32_t d, uint32_t a, uint32_t bt) {
            int kk = 0;
#pragma unroll
            for (int c = 0; c < T::NF; ++c)
#pragma unroll
                for (int k4 = 0; k4 < 4; ++k4, ++kk)
                    umma_f16_ss(d, smem_desc(a + c * 16384 + k4 * 32, 16, 1024, kSwizzle128),
                                smem_desc(bt + kk * 2048, T::T_TILE, 1024, kSwizzle128), id128, kk > 0);
            if (T::TAIL)
                umma_f16_ss(d, smem_desc(a + T::NF * 16384, 16, 256, kSwizzle32),
                            smem_desc(bt + kk * 2048, T::T_TILE, 1024, kSwizzle128), id128, 1);
        };
        auto issue_s = [&](int j) {
            const int b = j & 1;
            mbar_wait(&kf[b], (j >> 1) & 1);
            if (j >= 1) mbar_wait(s_empty, (j - 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                rows_x_t2(tmem + S_COL, smem_u32(sQ), smem_u32(sKt + b * KV_STAGE));
                umma_commit(s_full);
            }
            __syncwarp();
        };
        auto issue_dp = [&](int j) {
            const int b = j & 1;
            mbar_wait(&vf[b], (j >> 1) & 1);
            if (j >= 1) mbar_wait(dp_empty, (j - 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                rows_x_t2(tmem + DP_COL, smem_u32(sdO), smem_u32(sVt + b * KV_STAGE));
                umma_commit(dp_full);
                umma_commit(&ve[b]);  // V^T(j) is read by dP(j) only
            }
            __syncwarp();
        };
        mbar_wait(q_full, 0);
        if (nkv > 0) {
            issue_s(0);
            issue_dp(0);
        }
        for (int j = 0; j < nkv; ++j) {
            const int b = j & 1;
            if (j + 1 < nkv) issue_s(j + 1);
            mbar_wait(ds_full, j & 1);
            tc_fence_after();
            if (elect_one()) {  // dQ += dS_j K_j: 8 k-steps of 16 keys over the stage's two K^T tiles
                const uint32_t bt = smem_u32(sKt + b * KV_STAGE);
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    umma_f16_ts(tmem + DQ_COL, tmem + DS_COL + ks * 8,
                                smem_desc(bt + (ks >> 2) * T::T_TILE + (ks & 3) * 32, 16, 1024, kSwizzle128), idhd,
                                (j > 0 || ks > 0) ? 1u : 0u);
                umma_commit(dq_done);
                umma_commit(&ke[b]);  // K^T(j): S(j) and dQ(j) done
                if (j == nkv - 1) umma_commit(acc_done);
            }
            __syncwarp();
            if (j + 1 < nkv) issue_dp(j + 1);
        }
    } else if (warp >= 4) {
        // CW warps per TMEM lane group: warp hf handles keys [KW hf, KW hf + KW) of each step, 32 at a time
        const int g = warp & 3, hf = (warp - 4) >> 2, row = g * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(g * 32) << 16;
        const int q = q0 + row;
        const bool qv = q < f.Nq;
        const float lse2 = qv ? f.lse[(int64_t)h * lse_stride(f) + q] * kLog2e : 0.0f;
        const float Dq = qv ? p.Dvec[(int64_t)h * lse_stride(f) + q] : 0.0f;
        for (int j = 0; j < nkv; ++j) {
            float pr[KW];
            mbar_wait(s_full, j & 1);
            tc_fence_after();
#pragma unroll
            for (int u = 0; u < KW / 32; ++u)
                tmem_ld32(tmem + lane_base + S_COL + hf * KW + u * 32, reinterpret_cast<uint32_t*>(pr + 32 * u));
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(s_empty);
            const int kb = j * BKV + hf * KW;
            if (kb + KW <= f.Nk) {
#pragma unroll
                for (int c = 0; c < KW; ++c) pr[c] = ex2f(fmaf(pr[c], kLog2e, -lse2));
            } else {
#pragma unroll
                for (int c = 0; c < KW; ++c) pr[c] = kb + c < f.Nk ? ex2f(fmaf(pr[c], kLog2e, -lse2)) : 0.0f;
            }
            mbar_wait(dp_full, j & 1);
            tc_fence_after();
#pragma unroll
            for (int u = 0; u < KW / 32; ++u) {
                float dp[32];
                tmem_ld32(tmem + lane_base + DP_COL + hf * KW + u * 32, reinterpret_cast<uint32_t*>(dp));
                tmem_wait_ld();
                if (u == KW / 32 - 1) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(dp_empty);
                }
                uint32_t dk[16];
#pragma unroll
                for (int c = 0; c < 32; c += 2)
                    dk[c / 2] = pack_bf16(pr[32 * u + c] * (dp[c] - Dq), pr[32 * u + c + 1] * (dp[c + 1] - Dq));
                if (u == 0 && j >= 1) {
                    mbar_wait(dq_done, (j - 1) & 1);  // dQ(j-1) has read the dS columns
                    tc_fence_after();
                }
                tmem_st16(tmem + lane_base + DS_COL + hf * (KW / 2) + u * 16, dk);
            }
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(ds_full);
        }
        if (nkv > 0) mbar_wait(acc_done, 0);
        tc_fence_after();
        constexpr int NC = HD / 16;
        store_acc_row<HD>(tmem + lane_base + DQ_COL, static_cast<__nv_bfloat16*>(p.dq) + (int64_t)q * p.dq_ld + col,
                          qv && nkv > 0, hf * NC / CW, (hf + 1) * NC / CW);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

// =====================================================================================  dQ (v10)
// v9's 128-key steps with Q back in TMEM: S = Q K^T is a TS product, so the CTA's fixed A tile is no longer
// re-read from shared memory on every key step (v9's two SS products move 2 x 74 KB of shared memory per
// step, more than the tensor pipe's operand path sustains next to the TMA writes).  dS (bf16) is written over
// the consumed dP columns, which makes room for Q:  the compute warp that owns keys [64 hf, 64 hf + 64) has
// loaded all of its dP columns before it writes its dS pairs to [DP + 32 + 32 hf, +32), which lie inside its
// own dP range, and the pipe order dQ(j) -> dP(j+1) keeps the next dP behind the dS reader.  NS K^T / V^T
// stages (shared memory freed by Q).
// TMEM: S [0,128)  dP|dS [128,256)  dQ [256,256+HD)  Q (bf16 pairs) [400,472).
template <int HD, int NS>
__global__ void __launch_bounds__(128 + 128 * 2, 1) attn_bwd_dq_v10_kernel(const __grid_constant__ BwdMaps tm,
                                                                          AttnBwdProblem p) {
    constexpr int BMQ = 128, BKV = 128, CW = 2, KW = BKV / CW;
    using T = BT<HD>;
    constexpr int HDP = ((HD + 15) / 16) * 16;
    constexpr int S_COL = 0, DP_COL = 128, DS_COL = DP_COL + 32, DQ_COL = 256, Q_COL = 400;
    static_assert(DQ_COL + HDP <= Q_COL && Q_COL + HD / 2 <= 512, "TMEM budget");
    constexpr int KV_STAGE = 2 * T::T_TILE;  // two 64-key transposed tiles
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sdO = smem;
    uint8_t* sKt = sdO + T::ROW_TILE;    // [NS]
    uint8_t* sVt = sKt + NS * KV_STAGE;  // [NS]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sVt + NS * KV_STAGE);
    uint64_t* do_full = bars;
    uint64_t* kf = bars + 1;           // [NS]
    uint64_t* ke = kf + NS;            // [NS]
    uint64_t* vf = ke + NS;            // [NS]
    uint64_t* ve = vf + NS;            // [NS]
    uint64_t* s_full = ve + NS;
    uint64_t* s_empty = s_full + 1;
    uint64_t* dp_full = s_full + 2;
    uint64_t* ds_full = s_full + 3;
    uint64_t* acc_done = s_full + 4;
    uint64_t* qa_ready = s_full + 5;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 6);

    const AttnProblem& f = p.f;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int h = blockIdx.y, q0 = blockIdx.x * BMQ;
    const int nkv = (f.Nk + BKV - 1) / BKV;
    const int col = h * HD;

    if (threadIdx.x == 0) {
        mbar_init(do_full, 1);
        for (int i = 0; i < NS; ++i) {
            mbar_init(&kf[i], 1);
            mbar_init(&ke[i], 1);
            mbar_init(&vf[i], 1);
            mbar_init(&ve[i], 1);
        }
        mbar_init(s_full, 1);
        mbar_init(s_empty, 4 * CW);
        mbar_init(dp_full, 1);
        mbar_init(ds_full, 4 * CW);
        mbar_init(acc_done, 1);
        mbar_init(qa_ready, 4);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (elect_one()) {
            mbar_arrive_expect_tx(do_full, T::ROW_TILE);
            load_row_tile<HD>(sdO, &tm.b128, &tm.b32, do_full, col, q0);
            for (int j = 0; j < nkv; ++j) {
                const int b = j % NS;
                if (j >= NS) mbar_wait(&ke[b], ((j / NS) - 1) & 1);
                mbar_arrive_expect_tx(&kf[b], KV_STAGE);
                tma_load_2d(sKt + b * KV_STAGE, &tm.ta, &kf[b], j * BKV, col);
                tma_load_2d(sKt + b * KV_STAGE + T::T_TILE, &tm.ta, &kf[b], j * BKV + 64, col);
                if (j >= NS) mbar_wait(&ve[b], ((j / NS) - 1) & 1);
                mbar_arrive_expect_tx(&vf[b], KV_STAGE);
                tma_load_2d(sVt + b * KV_STAGE, &tm.tb, &vf[b], j * BKV, col);
                tma_load_2d(sVt + b * KV_STAGE + T::T_TILE, &tm.tb, &vf[b], j * BKV + 64, col);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t id128 = idesc_bf16_f32(128, 128, false, true), idhd = idesc_bf16_f32(128, HD, false, false);
        auto issue_s = [&](int j) {  // S = Q K^T: A = Q from TMEM, B^T = the stage's HD x 128 K^T tiles (MN-major)
            const int b = j % NS;
            mbar_wait(&kf[b], (j / NS) & 1);
            if (j >= 1) mbar_wait(s_empty, (j - 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t bt = smem_u32(sKt + b * KV_STAGE);
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk)
                    umma_f16_ts(tmem + S_COL, tmem + Q_COL + kk * 8, smem_desc(bt + kk * 2048, T::T_TILE, 1024, kSwizzle128),
                                id128, kk > 0 ? 1u : 0u);
                umma_commit(s_full);
            }
            __syncwarp();
        };
        auto issue_dp = [&](int j) {  // dP = dO V^T (SS); behind dQ(j-1) in the pipe, which has read dS(j-1)
            const int b = j % NS;
            mbar_wait(&vf[b], (j / NS) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t a = smem_u32(sdO), bt = smem_u32(sVt + b * KV_STAGE);
                int kk = 0;
#pragma unroll
                for (int c = 0; c < T::NF; ++c)
#pragma unroll
                    for (int k4 = 0; k4 < 4; ++k4, ++kk)
                        umma_f16_ss(tmem + DP_COL, smem_desc(a + c * 16384 + k4 * 32, 16, 1024, kSwizzle128),
                                    smem_desc(bt + kk * 2048, T::T_TILE, 1024, kSwizzle128), id128, kk > 0);
                if (T::TAIL)
                    umma_f16_ss(tmem + DP_COL, smem_desc(a + T::NF * 16384, 16, 256, kSwizzle32),
                                smem_desc(bt + kk * 2048, T::T_TILE, 1024, kSwizzle128), id128, 1);
                umma_commit(dp_full);
                umma_commit(&ve[b]);  // V^T(j) is read by dP(j) only
            }
            __syncwarp();
        };
        mbar_wait(qa_ready, 0);
        mbar_wait(do_full, 0);
        if (nkv > 0) {
            issue_s(0);
            issue_dp(0);
        }
        for (int j = 0; j < nkv; ++j) {
            const int b = j % NS;
            if (j + 1 < nkv) issue_s(j + 1);
            mbar_wait(ds_full, j & 1);
            tc_fence_after();
            if (elect_one()) {  // dQ += dS_j K_j: 8 k-steps of 16 keys over the stage's two K^T tiles
                const uint32_t bt = smem_u32(sKt + b * KV_STAGE);
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    umma_f16_ts(tmem + DQ_COL, tmem + DS_COL + ks * 8,
                                smem_desc(bt + (ks >> 2) * T::T_TILE + (ks & 3) * 32, 16, 1024, kSwizzle128), idhd,
                                (j > 0 || ks > 0) ? 1u : 0u);
                umma_commit(&ke[b]);  // K^T(j): S(j) and dQ(j) done
                if (j == nkv - 1) umma_commit(acc_done);
            }
            __syncwarp();
            if (j + 1 < nkv) issue_dp(j + 1);
        }
    } else if (warp >= 4) {
        // two warps per TMEM lane group: warp hf handles keys [64 hf, 64 hf + 64) of each step
        const int g = warp & 3, hf = (warp - 4) >> 2, row = g * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(g * 32) << 16;
        const int q = q0 + row;
        const bool qv = q < f.Nq;
        if (hf == 0) {
            row_to_tmem<HD>(tmem + lane_base + Q_COL,
                            static_cast<const __nv_bfloat16*>(f.q) + (int64_t)(qv ? q : 0) * f.q_ld + col, qv);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(qa_ready);
        }
        const float lse2 = qv ? f.lse[(int64_t)h * lse_stride(f) + q] * kLog2e : 0.0f;
        const float Dq = qv ? p.Dvec[(int64_t)h * lse_stride(f) + q] : 0.0f;
        for (int j = 0; j < nkv; ++j) {
            float pr[KW];
            mbar_wait(s_full, j & 1);
            tc_fence_after();
            tmem_ld32(tmem + lane_base + S_COL + hf * KW, reinterpret_cast<uint32_t*>(pr));
            tmem_ld32(tmem + lane_base + S_COL + hf * KW + 32, reinterpret_cast<uint32_t*>(pr + 32));
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(s_empty);
            const int kb = j * BKV + hf * KW;
            if (kb + KW <= f.Nk) {
#pragma unroll
                for (int c = 0; c < KW; ++c) pr[c] = ex2f(fmaf(pr[c], kLog2e, -lse2));
            } else {
#pragma unroll
                for (int c = 0; c < KW; ++c) pr[c] = kb + c < f.Nk ? ex2f(fmaf(pr[c], kLog2e, -lse2)) : 0.0f;
            }
            mbar_wait(dp_full, j & 1);
            tc_fence_after();
            float dp[KW];
            tmem_ld32(tmem + lane_base + DP_COL + hf * KW, reinterpret_cast<uint32_t*>(dp));
            tmem_ld32(tmem + lane_base + DP_COL + hf * KW + 32, reinterpret_cast<uint32_t*>(dp + 32));
            tmem_wait_ld();  // all of this warp's dP columns are in registers before its dS overwrites them
            uint32_t dk[KW / 2];
#pragma unroll
            for (int c = 0; c < KW; c += 2)
                dk[c / 2] = pack_bf16(pr[c] * (dp[c] - Dq), pr[c + 1] * (dp[c + 1] - Dq));  // autodiff.cpp:820
            tmem_st16(tmem + lane_base + DS_COL + hf * (KW / 2), dk);
            tmem_st16(tmem + lane_base + DS_COL + hf * (KW / 2) + 16, dk + 16);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(ds_full);
        }
        if (nkv > 0) mbar_wait(acc_done, 0);
        tc_fence_after();
        constexpr int NC = HD / 16;
        store_acc_row<HD>(tmem + lane_base + DQ_COL, static_cast<__nv_bfloat16*>(p.dq) + (int64_t)q * p.dq_ld + col,
                          qv && nkv > 0, hf * NC / CW, (hf + 1) * NC / CW);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ host
template <int HD>
static void launch_bwd(const AttnBwdProblem& p, const void* qt, int64_t qt_ld, const void* kt, int64_t kt_ld,
                       const void* vt, int64_t vt_ld, const void* dot, int64_t dot_ld, cudaStream_t s) {
    using T = BT<HD>;
    const AttnProblem& f = p.f;
    const uint64_t W = (uint64_t)f.heads * HD;
    attn_bwd_dvec(p, s);
    {
        BwdMaps m;
        if (reinterpret_cast<uintptr_t>(f.k) % 16 || f.k_ld % 8)
            throw std::runtime_error("attn_bwd_tc: k must be 16-byte aligned with ld % 8 == 0");
        make_tmap_sw(&m.b128, f.v, W, f.Nk, f.v_ld, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
        make_tmap_sw(&m.b32, f.v, W, f.Nk, f.v_ld, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B);
        make_tmap_sw(&m.a128, f.k, W, f.Nk, f.k_ld, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
        make_tmap_sw(&m.a32, f.k, W, f.Nk, f.k_ld, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B);
        make_tmap_sw(&m.ta, qt, f.Nq, W, qt_ld, 64, HD, CU_TENSOR_MAP_SWIZZLE_128B);
        make_tmap_sw(&m.tb, dot, f.Nq, W, dot_ld, 64, HD, CU_TENSOR_MAP_SWIZZLE_128B);
        const int smem = T::ROW_TILE + 10 * T::T_TILE + 10 * 64 * 4 + 256 + 1024;
        const int smem8 = smem + (HD > 128 ? 4096 : 0);
        static bool set = false;
        if (!set) {
            MGV_CUDA(cudaFuncSetAttribute(attn_bwd_dkv_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            MGV_CUDA(cudaFuncSetAttribute(attn_bwd_dkv_v8_kernel<HD, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          smem8));
            MGV_CUDA(cudaFuncSetAttribute(attn_bwd_dkv_v8_kernel<HD, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          smem8));
            set = true;
        }
        // few key tiles (cross-attention): split the query range so the grid still covers the SMs
        const int kv_ctas = (f.Nk + 127) / 128 * f.heads, nq_all = (f.Nq + 63) / 64;
        const int splits = std::max(1, std::min({num_sms() / std::max(kv_ctas, 1), nq_all / 8, 16}));
        float* part = nullptr;
        if (splits > 1) MGV_CUDA(cudaMallocAsync(&part, sizeof(float) * splits * f.Nk * 2 * W, s));
        if (splits == 1 && g_dkv_variant == 2) {
            // v9: CTA pairs over 256 keys, M = 256 UMMAs (the operand tiles split as described at the kernel)
            using PT = PairT<HD>;
            BwdMaps m2;
            if ((reinterpret_cast<uintptr_t>(f.q) | reinterpret_cast<uintptr_t>(p.dO)) % 16 || f.q_ld % 8 || p.do_ld % 8)
                throw std::runtime_error("attn_bwd_tc: q / dO must be 16-byte aligned with ld % 8 == 0");
            make_tmap_sw(&m2.a128, f.q, W, f.Nq, f.q_ld, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B);
            make_tmap_sw(&m2.a32, f.q, W, f.Nq, f.q_ld, 16, 32, CU_TENSOR_MAP_SWIZZLE_32B);
            make_tmap_sw(&m2.b128, p.dO, W, f.Nq, p.do_ld, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B);
            make_tmap_sw(&m2.b32, p.dO, W, f.Nq, p.do_ld, 16, 32, CU_TENSOR_MAP_SWIZZLE_32B);
            make_tmap_sw(&m2.ta, qt, f.Nq, W, qt_ld, 64, PT::HH, CU_TENSOR_MAP_SWIZZLE_128B);
            make_tmap_sw(&m2.tb, dot, f.Nq, W, dot_ld, 64, PT::HH, CU_TENSOR_MAP_SWIZZLE_128B);
            const int psmem = T::ROW_TILE + (HD > 128 ? 4096 : 0) + 5 * PT::STAGE + 10 * 64 * 4 + 256 + 1024;
            static bool pset9 = false;
            if (!pset9) {
                MGV_CUDA(cudaFuncSetAttribute(attn_bwd_dkv_v9_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              psmem));
                pset9 = true;
            }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(2 * ((f.Nk + 255) / 256), f.heads);
            cfg.blockDim = dim3(384);
            cfg.dynamicSmemBytes = psmem;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 2;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            MGV_CUDA(cudaLaunchKernelEx(&cfg, attn_bwd_dkv_v9_kernel<HD>, m, m2, p));
        } else if (splits == 1 && g_dkv_pair) {
            // one 2-CTA cluster per key tile (head_dim split over the pair, P^T / dS^T exchanged via DSMEM)
            const int psmem = 8 * T::T_TILE + 4 * 128 * 64 * 2 + 4 * 64 * 4 + 256 + 1024;
            static bool pset = false;
            if (!pset) {
                MGV_CUDA(cudaFuncSetAttribute(attn_bwd_dkv_pair_kernel<HD>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, psmem));
                pset = true;
            }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(2 * ((f.Nk + 127) / 128), f.heads);
            cfg.blockDim = dim3(384);
            cfg.dynamicSmemBytes = psmem;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 2;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            MGV_CUDA(cudaLaunchKernelEx(&cfg, attn_bwd_dkv_pair_kernel<HD>, m, p));
        } else {
            if (g_dkv_variant == 1)
                attn_bwd_dkv_tc_kernel<HD><<<dim3((f.Nk + 127) / 128, f.heads, splits), 384, smem, s>>>(m, p, part);
            else
                if (g_dkv_cw == 4)
                    attn_bwd_dkv_v8_kernel<HD, 4><<<dim3((f.Nk + 127) / 128, f.heads, splits), 640, smem8, s>>>(m, p,
                                                                                                          part);
                else
                    attn_bwd_dkv_v8_kernel<HD, 2><<<dim3((f.Nk + 127) / 128, f.heads, splits), 384, smem8, s>>>(m, p,
                                                                                                          part);
        }
        ::mgv::note_launch();
        MGV_CUDA(cudaGetLastError());
        if (splits > 1) {
            const int64_t n = (int64_t)f.Nk * 2 * W;
            reduce_dkv_parts<<<static_cast<int>(std::min<int64_t>((n + 255) / 256, 4096)), 256, 0, s>>>(
                part, splits, f.Nk, W, static_cast<__nv_bfloat16*>(p.dv), p.dv_ld, static_cast<__nv_bfloat16*>(p.dk),
                p.dk_ld);
            ::mgv::note_launch();
            MGV_CUDA(cudaGetLastError());
            MGV_CUDA(cudaFreeAsync(part, s));
        }
    }
    {
        BwdMaps m;
        make_tmap_sw(&m.ta, kt, f.Nk, W, kt_ld, 64, HD, CU_TENSOR_MAP_SWIZZLE_128B);
        make_tmap_sw(&m.tb, vt, f.Nk, W, vt_ld, 64, HD, CU_TENSOR_MAP_SWIZZLE_128B);
        // Q / dO rows are read straight into TMEM with 16-byte loads
        if ((reinterpret_cast<uintptr_t>(f.q) | reinterpret_cast<uintptr_t>(p.dO)) % 16 || f.q_ld % 8 || p.do_ld % 8)
            throw std::runtime_error("attn_bwd_tc: q / dO must be 16-byte aligned with ld % 8 == 0");
        const int smem = 12 * T::T_TILE + 256 + 1024;
        static bool set = false;
        if (!set) {
            MGV_CUDA(cudaFuncSetAttribute(attn_bwd_dq_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            set = true;
        }
        if (g_dq_variant == 3) {  // v10: 128-key steps, Q in TMEM, dO in shared memory, dS over dP
            make_tmap_sw(&m.b128, p.dO, W, f.Nq, p.do_ld, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
            make_tmap_sw(&m.b32, p.dO, W, f.Nq, p.do_ld, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B);
            const int smem10 = T::ROW_TILE + 8 * T::T_TILE + 256 + 1024;
            static bool set10 = false;
            if (!set10) {
                MGV_CUDA(cudaFuncSetAttribute(attn_bwd_dq_v10_kernel<HD, 2>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, smem10));
                set10 = true;
            }
            attn_bwd_dq_v10_kernel<HD, 2><<<dim3((f.Nq + 127) / 128, f.heads), 128 + 128 * 2, smem10, s>>>(m, p);
        } else if (g_dq_variant == 2) {  // v9: 128-key steps, Q and dO in shared memory
            make_tmap_sw(&m.a128, f.q, W, f.Nq, f.q_ld, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
            make_tmap_sw(&m.a32, f.q, W, f.Nq, f.q_ld, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B);
            make_tmap_sw(&m.b128, p.dO, W, f.Nq, p.do_ld, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
            make_tmap_sw(&m.b32, p.dO, W, f.Nq, p.do_ld, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B);
            const int smem9 = 2 * T::ROW_TILE + 8 * T::T_TILE + 256 + 1024;
            static bool set9 = false;
            if (!set9) {
                MGV_CUDA(cudaFuncSetAttribute(attn_bwd_dq_v9_kernel<HD, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              smem9));
                MGV_CUDA(cudaFuncSetAttribute(attn_bwd_dq_v9_kernel<HD, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              smem9));
                set9 = true;
            }
            if (g_dq_cw == 4)
                attn_bwd_dq_v9_kernel<HD, 4><<<dim3((f.Nq + 127) / 128, f.heads), 128 + 128 * 4, smem9, s>>>(m, p);
            else
                attn_bwd_dq_v9_kernel<HD, 2><<<dim3((f.Nq + 127) / 128, f.heads), 128 + 128 * 2, smem9, s>>>(m, p);
        } else if (g_dq_variant == 1) {  // v8: Q in shared memory, dP double-buffered
            make_tmap_sw(&m.a128, f.q, W, f.Nq, f.q_ld, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
            make_tmap_sw(&m.a32, f.q, W, f.Nq, f.q_ld, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B);
            const int smem8 = T::ROW_TILE + 10 * T::T_TILE + 256 + 1024;
            static bool set8 = false;
            if (!set8) {
                MGV_CUDA(cudaFuncSetAttribute(attn_bwd_dq_v8_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              smem8));
                set8 = true;
            }
            attn_bwd_dq_v8_kernel<HD><<<dim3((f.Nq + 127) / 128, f.heads), 128 + 128 * kCWq, smem8, s>>>(m, p);
        } else {
            attn_bwd_dq_tc_kernel<HD><<<dim3((f.Nq + 127) / 128, f.heads), 128 + 128 * kCWq, smem, s>>>(m, p);
        }
        ::mgv::note_launch();
        MGV_CUDA(cudaGetLastError());
    }
}

void attn_bwd_tc(const AttnBwdProblem& p, cudaStream_t s) {
    const AttnProblem& f = p.f;
    const int W = f.heads * f.hd;
    // transposed operands: use the caller's, else make them here
    std::vector<__nv_bfloat16*> tmp;
    auto make_t = [&](const void* src, int64_t ld, int rows, int64_t* out_ld) -> const void* {
        const int64_t l = (rows + 7) / 8 * 8;
        __nv_bfloat16* d = nullptr;
        MGV_CUDA(cudaMallocAsync(&d, sizeof(__nv_bfloat16) * l * W, s));
        transpose_bf16(static_cast<const __nv_bfloat16*>(src), ld, rows, W, d, l, s);
        tmp.push_back(d);
        *out_ld = l;
        return d;
    };
    int64_t qt_ld = p.qt_ld, kt_ld = p.kt_ld, vt_ld = f.vt_ld, dot_ld = p.dot_ld;
    const void* qt = p.qt ? p.qt : make_t(f.q, f.q_ld, f.Nq, &qt_ld);
    const void* kt = p.kt ? p.kt : make_t(f.k, f.k_ld, f.Nk, &kt_ld);
    const void* vt = f.vt ? f.vt : make_t(f.v, f.v_ld, f.Nk, &vt_ld);
    const void* dot = p.dot ? p.dot : make_t(p.dO, p.do_ld, f.Nq, &dot_ld);
    // lse / D rows are streamed with bulk copies: per-head stride must be a multiple of 64 covering Nq
    AttnBwdProblem q = p;
    const int64_t need = (static_cast<int64_t>(f.Nq) + 63) / 64 * 64;
    std::vector<float*> ftmp;
    if (lse_stride(f) < need || lse_stride(f) % 64 != 0) {
        float *lse = nullptr, *dv = nullptr;
        MGV_CUDA(cudaMallocAsync(&lse, sizeof(float) * need * f.heads, s));
        MGV_CUDA(cudaMallocAsync(&dv, sizeof(float) * need * f.heads, s));
        MGV_CUDA(cudaMemcpy2DAsync(lse, need * sizeof(float), f.lse, lse_stride(f) * sizeof(float),
                                   f.Nq * sizeof(float), f.heads, cudaMemcpyDeviceToDevice, s));
        q.f.lse = lse;
        q.f.lse_ld = need;
        q.Dvec = dv;
        ftmp = {lse, dv};
    }
    switch (f.hd) {
        case 64: launch_bwd<64>(q, qt, qt_ld, kt, kt_ld, vt, vt_ld, dot, dot_ld, s); break;
        case 128: launch_bwd<128>(q, qt, qt_ld, kt, kt_ld, vt, vt_ld, dot, dot_ld, s); break;
        case 144: launch_bwd<144>(q, qt, qt_ld, kt, kt_ld, vt, vt_ld, dot, dot_ld, s); break;
        default: throw std::runtime_error("attn_bwd_tc: unsupported head_dim");
    }
    for (auto* d : tmp) MGV_CUDA(cudaFreeAsync(d, s));
    for (auto* d : ftmp) MGV_CUDA(cudaFreeAsync(d, s));
}

}  // namespace mgv

#ifdef MGV_ATTN_TRACE
extern "C" int mgv_dev_attn_trace(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, mgv::g_attn_trace, sizeof(mgv::g_attn_trace)) == cudaSuccess ? 0 : 1;
}
extern "C" int mgv_dev_attn_trace2(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, mgv::g_attn_trace2, sizeof(mgv::g_attn_trace2)) == cudaSuccess ? 0 : 1;
}
#endif

extern "C" int mgv_dev_set_dkv_pair(int on) {
    mgv::g_dkv_pair = on ? 1 : 0;
    return 0;
}
extern "C" int mgv_dev_set_attn_dbg(int v) {
    return cudaMemcpyToSymbol(mgv::g_attn_dbg, &v, sizeof(int)) == cudaSuccess ? 0 : 1;
}
extern "C" int mgv_dev_set_dq_variant(int v) {
    mgv::g_dq_variant = v % 10;
    mgv::g_dq_cw = v >= 10 ? 4 : 2;  // 12: v9 with 4 compute warps per lane group
    return 0;
}
extern "C" int mgv_dev_set_dkv_variant(int v) {
    mgv::g_dkv_variant = v % 10;
    mgv::g_dkv_cw = v >= 10 ? 4 : 2;  // 10: v8 with 4 compute warps per lane group
    return 0;
}

// diagnostics: how many 2-CTA clusters of the dK/dV pair kernel can be resident at once (head_dim 144)
extern "C" int mgv_dev_dkv_pair_clusters() {
    using T = mgv::BT<144>;
    const int psmem = 8 * T::T_TILE + 4 * 128 * 64 * 2 + 4 * 64 * 4 + 256 + 1024;
    cudaFuncSetAttribute(mgv::attn_bwd_dkv_pair_kernel<144>, cudaFuncAttributeMaxDynamicSharedMemorySize, psmem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * 450, 24);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = psmem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = -1;
    if (cudaOccupancyMaxActiveClusters(&n, mgv::attn_bwd_dkv_pair_kernel<144>, &cfg) != cudaSuccess) return -1;
    return n;
}
