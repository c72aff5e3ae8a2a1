// tcgen05 flash-attention backward for sm_100a, deterministic (no atomics):
// the gradient of Tape::mha (autodiff.cpp:795-843) in two passes.
//
//   dK/dV pass  CTA per (128-key tile, head), loops over 128-query steps:
//                 S^T = K Q^T,  dP^T = V dO^T          (SS; Q^T/dO^T tiles read MN-major)
//                 P^T = exp(S^T - lse), dS^T = P^T (dP^T - D)   (thread = key row)
//                 dV += P^T dO, dK += dS^T Q           (TS; dO^T/Q^T read K-major, one N = hd MMA per k-step)
//   dQ pass     CTA per (128-query tile, head), loops over 128-key steps:
//                 S = Q K^T (TS), dP = dO V^T (SS)
//                 dS = P (dP - D)                      (thread = query row)
//                 dQ += dS K                           (TS; K^T tiles read K-major, N = hd)
// The transposed operands (Q^T, K^T, V^T, dO^T: [heads*hd][tokens]) are made
// once per step by a tiled transpose, so no MMA ever splits head_dim 144 into
// 128 + 16.  The MMA warp issues the next tile's products under the current
// tile's elementwise work.  Earlier variants (64-query dK/dV steps with V in TMEM,
// CTA-pair / DSMEM exchanges, 64-key dQ steps) are in the history of this file.
#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <vector>

#include "attn.h"
#include "gemm.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace mgv {


namespace {

constexpr float kLog2e = 1.4426950408889634f;

// Timing experiments of the dK/dV pass (wrong results; tools/build_variant.sh, never in the product build):
//   1: no Q^T / dO^T TMA after the first stages (the resident tiles are reused)
//   2: no exponentials (P = S)      4: compute warps skip all TMEM loads / stores (they only bounce barriers)
#ifndef MGV_DKV_X
#define MGV_DKV_X 0
#endif
// dQ pass timing experiment: MGV_DQ_X 2 = no exponentials
#ifndef MGV_DQ_X
#define MGV_DQ_X 0
#endif

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

__device__ __forceinline__ float4 lds_f4(uint32_t saddr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(saddr));
    return v;
}

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

// =====================================================================================  dK / dV (v11)
// 128-query steps with every product an N >= 128 MMA (34 instructions per 128 queries, against 52 for the
// 64-query-step pass it replaced).  TMEM:
//   SD [0,128)    S^T(i) -> (loaded into registers) -> dP^T(i) -> (loaded) -> S^T(i+1)
//   PT [128,192)  P^T(i) (bf16 pairs) -> (read by dV(i)) -> dS^T(i) -> (read by dK(i)) -> P^T(i+1)
//   dV [192, 192+HDP)   dK [.., +HDP)
// MMA issue order per step:  dP^T(i) [S^T(i) loaded]  dV(i) [P^T(i) stored]  S^T(i+1) [dP^T(i) loaded]
// dK(i) [dS^T(i) stored]; the in-order tensor pipe keeps each overwrite behind its reader.  Operands:
//   S^T  = K Q^T    SS: K row tile (K-major) x two 64-token Q^T tiles read MN-major (LBO = one tile)
//   dP^T = V dO^T   SS: V row tile x the dO^T tiles, MN-major
//   dV  += P^T dO   TS: P^T from TMEM x the dO^T tiles read K-major (N = HD)
//   dK  += dS^T Q   TS: dS^T from TMEM x the Q^T tiles read K-major
// The exponentials of step i run under dK(i-1) and dP^T(i); dS(i) under S^T(i+1).
template <int HD>
__device__ __forceinline__ void mma_rows_x_t128(uint32_t d, uint32_t a, uint32_t bt) {
    using T = BT<HD>;
    constexpr uint32_t id = idesc_bf16_f32(128, 128, false, true);
    int kk = 0;
#pragma unroll
    for (int c = 0; c < T::NF; ++c)
#pragma unroll
        for (int k = 0; k < 4; ++k, ++kk)
            umma_f16_ss(d, smem_desc(a + c * 16384 + k * 32, 16, 1024, kSwizzle128),
                        smem_desc(bt + kk * 2048, T::T_TILE, 1024, kSwizzle128), id, kk > 0);
    if (T::TAIL)
        umma_f16_ss(d, smem_desc(a + T::NF * 16384, 16, 256, kSwizzle32),
                    smem_desc(bt + kk * 2048, T::T_TILE, 1024, kSwizzle128), id, 1);
}
// D[128 x HD] (+)= A[128 x 128] (TMEM, bf16 pairs, 64 columns) . B with B two HD x 64 transposed tiles read
// K-major (K = 128 tokens): eight N = HD MMAs
template <int HD>
__device__ __forceinline__ void mma_tmem128_x_t(uint32_t d, uint32_t a_tmem, uint32_t bt, bool acc_first) {
    using T = BT<HD>;
    constexpr uint32_t id = idesc_bf16_f32(128, HD, false, false);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)
        umma_f16_ts(d, a_tmem + ks * 8, smem_desc(bt + (ks >> 2) * T::T_TILE + (ks & 3) * 32, 16, 1024, kSwizzle128),
                    id, (acc_first || ks > 0) ? 1u : 0u);
}

// CW: compute warps per TMEM lane group (each owns 128 / CW query columns of a step).  CW = 4 (640 threads, 95
// registers) measured 71.6 ms against 70.3 for CW = 2 at 57,600 tokens (profiles/r02/attn_bwd_cw_poly_r02.log)
template <int HD, int CW>
__global__ void __launch_bounds__(128 + 128 * CW, 1) attn_bwd_dkv_v11_kernel(const __grid_constant__ BwdMaps tm,
                                                                           AttnBwdProblem p, float* part) {
    constexpr int BKV = 128, BQ = 128, NST = 2, QW = BQ / CW;
    static_assert(CW == 2 || CW == 4, "2 or 4 compute warps per lane group");
    using T = BT<HD>;
    constexpr int HDP = ((HD + 15) / 16) * 16;
    constexpr int SD_COL = 0, PT_COL = 128, DV_COL = 192, DK_COL = DV_COL + HDP;
    static_assert(DK_COL + HDP <= 512, "TMEM budget");
    constexpr int QT = 2 * T::T_TILE;  // 128 tokens of a transposed operand (two 64-token tiles)
    constexpr int ROW_BYTES = T::NF * 16384 + (T::TAIL ? 4096 : 0);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sK = smem;
    uint8_t* sV = sK + T::ROW_TILE;
    uint8_t* sQt = sV + T::ROW_TILE;   // [NST]
    uint8_t* sdOt = sQt + NST * QT;     // [NST]
    float* sLse = reinterpret_cast<float*>(sdOt + NST * QT);  // [NST][BQ]
    float* sD = sLse + NST * BQ;                               // [NST][BQ]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sD + NST * BQ);
    uint64_t* k_full = bars;
    uint64_t* qd_full = bars + 1;         // [NST]
    uint64_t* qd_empty = bars + 1 + NST;  // [NST]
    uint64_t* s_full = bars + 1 + 2 * NST;
    uint64_t* s_loaded = s_full + 1;
    uint64_t* dp_full = s_full + 2;
    uint64_t* dp_loaded = s_full + 3;
    uint64_t* p_full = s_full + 4;
    uint64_t* pv_done = s_full + 5;
    uint64_t* ds_full = s_full + 6;
    uint64_t* dk_done = s_full + 7;
    uint64_t* acc_done = s_full + 8;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 9);

    const AttnProblem& f = p.f;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int h = blockIdx.y, k0 = blockIdx.x * BKV;
    // packed segments (AttnProblem::seg): this key tile's segment [qlo, qend) is also its query range; keys at or
    // past qend are padding rows (their dK / dV rows are written as zeros)
    const int qlo = f.seg ? f.seg[2 * (k0 / 128)] : 0, qend = f.seg ? f.seg[2 * (k0 / 128) + 1] : f.Nq;
    const int kend = f.seg ? qend : f.Nk;
    const int nq_all = (qend - qlo + BQ - 1) / BQ;
    const int i0 = qlo / BQ + static_cast<int>((int64_t)blockIdx.z * nq_all / gridDim.z);
    const int nq = static_cast<int>((int64_t)(blockIdx.z + 1) * nq_all / gridDim.z) -
                   static_cast<int>((int64_t)blockIdx.z * nq_all / gridDim.z);  // this split's steps
    const int col = h * HD;

    if (threadIdx.x == 0) {
        mbar_init(k_full, 1);
        for (int i = 0; i < NST; ++i) {
            mbar_init(&qd_full[i], 1);
            mbar_init(&qd_empty[i], 1);
        }
        mbar_init(s_full, 1);
        mbar_init(s_loaded, 4 * CW);
        mbar_init(dp_full, 1);
        mbar_init(dp_loaded, 4 * CW);
        mbar_init(p_full, 4 * CW);
        mbar_init(pv_done, 1);
        mbar_init(ds_full, 4 * CW);
        mbar_init(dk_done, 1);
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
            mbar_arrive_expect_tx(k_full, 2 * ROW_BYTES);
            load_row_tile<HD>(sK, &tm.a128, &tm.a32, k_full, col, k0);
            load_row_tile<HD>(sV, &tm.b128, &tm.b32, k_full, col, k0);
            for (int i = 0; i < nq; ++i) {
                const int st = i % NST;
                if (i >= NST) mbar_wait(&qd_empty[st], ((i / NST) - 1) & 1);
                if ((MGV_DKV_X & 1) && i >= NST) {
                    mbar_arrive(&qd_full[st]);
                    continue;
                }
                mbar_arrive_expect_tx(&qd_full[st], 2 * QT + 2 * BQ * 4);
                const int qt = (i0 + i) * BQ;
                tma_load_2d(sQt + st * QT, &tm.ta, &qd_full[st], qt, col);
                tma_load_2d(sQt + st * QT + T::T_TILE, &tm.ta, &qd_full[st], qt + 64, col);
                tma_load_2d(sdOt + st * QT, &tm.tb, &qd_full[st], qt, col);
                tma_load_2d(sdOt + st * QT + T::T_TILE, &tm.tb, &qd_full[st], qt + 64, col);
                bulk_load(sLse + st * BQ, f.lse + (int64_t)h * lse_stride(f) + qt, BQ * 4, &qd_full[st]);
                bulk_load(sD + st * BQ, p.Dvec + (int64_t)h * lse_stride(f) + qt, BQ * 4, &qd_full[st]);
            }
        }
    } else if (warp == 1) {
        const uint32_t aK = smem_u32(sK), aV = smem_u32(sV);
        mbar_wait(k_full, 0);
        if (nq > 0) {
            mbar_wait(&qd_full[0], 0);
            tc_fence_after();
            if (elect_one()) {
                mma_rows_x_t128<HD>(tmem + SD_COL, aK, smem_u32(sQt));
                umma_commit(s_full);
            }
            __syncwarp();
        }
        for (int i = 0; i < nq; ++i) {
            const int st = i % NST;
            mbar_wait(s_loaded, i & 1);  // S^T(i) is in registers: dP^T(i) may overwrite it
            tc_fence_after();
            if (lane == 0) ATR8(0, i);
            if (elect_one()) {
                mma_rows_x_t128<HD>(tmem + SD_COL, aV, smem_u32(sdOt + st * QT));
                umma_commit(dp_full);
            }
            __syncwarp();
            mbar_wait(p_full, i & 1);
            tc_fence_after();
            if (lane == 0) ATR8(1, i);
            if (elect_one()) {
                mma_tmem128_x_t<HD>(tmem + DV_COL, tmem + PT_COL, smem_u32(sdOt + st * QT), i > 0);
                umma_commit(pv_done);
            }
            __syncwarp();
            if (i + 1 < nq) {
                mbar_wait(dp_loaded, i & 1);  // dP^T(i) is in registers: S^T(i+1) may overwrite it
                mbar_wait(&qd_full[(i + 1) % NST], ((i + 1) / NST) & 1);
                tc_fence_after();
                if (lane == 0) ATR8(2, i);
                if (elect_one()) {
                    mma_rows_x_t128<HD>(tmem + SD_COL, aK, smem_u32(sQt + ((i + 1) % NST) * QT));
                    umma_commit(s_full);
                }
                __syncwarp();
            }
            mbar_wait(ds_full, i & 1);
            tc_fence_after();
            if (lane == 0) ATR8(3, i);
            if (elect_one()) {
                mma_tmem128_x_t<HD>(tmem + DK_COL, tmem + PT_COL, smem_u32(sQt + st * QT), i > 0);
                umma_commit(dk_done);
                umma_commit(&qd_empty[st]);
                if (i == nq - 1) umma_commit(acc_done);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        // CW warps per TMEM lane group: warp hf owns query columns [QW hf, QW hf + QW) of each step
        const int g = warp & 3, hf = (warp - 4) >> 2, row = g * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(g * 32) << 16;
        const int kv = k0 + row;
        const bool kvv = kv < f.Nk, kreal = kv < kend;
        const uint32_t sd = tmem + lane_base + SD_COL + hf * QW, pt = tmem + lane_base + PT_COL + hf * (QW / 2);
        for (int i = 0; i < nq; ++i) {
            const int st = i % NST;
            mbar_wait(&qd_full[st], (i / NST) & 1);  // lse / D rows of this step have landed
            mbar_wait(s_full, i & 1);
            tc_fence_after();
            if (warp == 4 && lane == 0) ATR8(4, i);
            float s[QW];
            if (!(MGV_DKV_X & 4)) {
#pragma unroll
                for (int c = 0; c < QW; c += 32) tmem_ld32(sd + c, reinterpret_cast<uint32_t*>(s + c));
                tmem_wait_ld();
            } else {
#pragma unroll
                for (int c = 0; c < QW; ++c) s[c] = __int_as_float(lane + c);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(s_loaded);
            // lse / D rows: 16-byte shared-memory broadcasts (one wavefront per 4 queries per warp); per-element
            // generic loads made the compute warps' shared wavefronts outnumber the SS MMAs' operand reads
            const uint32_t lse_s = smem_u32(sLse + st * BQ + hf * QW), d_s = smem_u32(sD + st * BQ + hf * QW);
            const int qb = (i0 + i) * BQ + hf * QW;
            const bool full = qb + QW <= qend;
            uint32_t pk[QW / 2];
            const float2 lg2 = make_float2(kLog2e, kLog2e);
            if (full) {  // warp-uniform: no per-column masking; packed f32x2 arithmetic (bit-identical to scalar)
#pragma unroll
                for (int c4 = 0; c4 < QW; c4 += 4) {
                    const float4 l = lds_f4(lse_s + c4 * 4);
                    const float2 x0 = fmul2(fsub2(make_float2(s[c4], s[c4 + 1]), make_float2(l.x, l.y)), lg2);
                    const float2 x1 = fmul2(fsub2(make_float2(s[c4 + 2], s[c4 + 3]), make_float2(l.z, l.w)), lg2);
                    if (MGV_DKV_X & 2) {
                        s[c4] = x0.x;
                        s[c4 + 1] = x0.y;
                        s[c4 + 2] = x1.x;
                        s[c4 + 3] = x1.y;
                    } else {
                        s[c4] = ex2f(x0.x);
                        s[c4 + 1] = ex2f(x0.y);
                        s[c4 + 2] = ex2f(x1.x);
                        s[c4 + 3] = ex2f(x1.y);
                    }
                    pk[c4 / 2] = pack_bf16(s[c4], s[c4 + 1]);
                    pk[c4 / 2 + 1] = pack_bf16(s[c4 + 2], s[c4 + 3]);
                }
            } else {
#pragma unroll
                for (int c4 = 0; c4 < QW; c4 += 4) {
                    const float4 l = lds_f4(lse_s + c4 * 4);
                    const float lv[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int c = c4 + e;
                        s[c] = qb + c < qend ? ex2f((s[c] - lv[e]) * kLog2e) : 0.0f;  // lse rows are natural-log
                    }
                    pk[c4 / 2] = pack_bf16(s[c4], s[c4 + 1]);
                    pk[c4 / 2 + 1] = pack_bf16(s[c4 + 2], s[c4 + 3]);
                }
            }
            if (i >= 1) {
                mbar_wait(dk_done, (i - 1) & 1);  // dK(i-1) has read dS^T(i-1) out of PT
                tc_fence_after();
            }
            if (!(MGV_DKV_X & 4)) {
                if constexpr (QW == 64)
                    tmem_st32(pt, pk);
                else
                    tmem_st16(pt, pk);
                tmem_wait_st();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(p_full);
            if (warp == 4 && lane == 0) ATR8(5, i);
            mbar_wait(dp_full, i & 1);
            tc_fence_after();
            if (warp == 4 && lane == 0) ATR8(6, i);
            float dp[QW];
            if (!(MGV_DKV_X & 4)) {
#pragma unroll
                for (int c = 0; c < QW; c += 32) tmem_ld32(sd + c, reinterpret_cast<uint32_t*>(dp + c));
                tmem_wait_ld();
            } else {
#pragma unroll
                for (int c = 0; c < QW; ++c) dp[c] = s[c];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(dp_loaded);  // S^T(i+1) may now overwrite SD, under the dS math below
#pragma unroll
            for (int c = 0; c < QW; c += 4) {  // dS = P (dP - D) (autodiff.cpp:820), packed pairs
                const float4 dd = lds_f4(d_s + c * 4);
                const float2 d0 = fmul2(make_float2(s[c], s[c + 1]),
                                        fsub2(make_float2(dp[c], dp[c + 1]), make_float2(dd.x, dd.y)));
                const float2 d1 = fmul2(make_float2(s[c + 2], s[c + 3]),
                                        fsub2(make_float2(dp[c + 2], dp[c + 3]), make_float2(dd.z, dd.w)));
                pk[c / 2] = pack_bf16(d0.x, d0.y);
                pk[c / 2 + 1] = pack_bf16(d1.x, d1.y);
            }
            mbar_wait(pv_done, i & 1);  // dV(i) has read P^T(i) out of PT
            tc_fence_after();
            if (warp == 4 && lane == 0) ATR8(7, i);
            if (!(MGV_DKV_X & 4)) {
                if constexpr (QW == 64)
                    tmem_st32(pt, pk);
                else
                    tmem_st16(pt, pk);
                tmem_wait_st();
            } else if (pk[0] == 0x12345678u && pk[QW / 2 - 1] == 0x9abcdef0u) {
                p.dv = nullptr;  // keeps the math alive in the experiment build
            }
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
            const int part_i = is_v ? hf : hf - HALF, c0 = part_i * NC / HALF, c1 = (part_i + 1) * NC / HALF;
            __nv_bfloat16* out = is_v ? static_cast<__nv_bfloat16*>(p.dv) + (int64_t)kv * p.dv_ld + col
                                      : static_cast<__nv_bfloat16*>(p.dk) + (int64_t)kv * p.dk_ld + col;
            // every lane runs the (warp-collective) TMEM loads; a padding key row of a packed segment stores zeros
            store_acc_row<HD>(tmem + lane_base + (is_v ? DV_COL : DK_COL), out, valid && kreal, c0, c1);
            if (valid && !kreal) {
                const uint4 z = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll 1
                for (int c = 2 * c0; c < 2 * c1; ++c) reinterpret_cast<uint4*>(out)[c] = z;
            }
        }
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
template <int HD, int NS>  // NS: K^T stages (V^T: 2; V^T is released by dP, K^T only by dQ)
__global__ void __launch_bounds__(128 + 128 * 2, 1) attn_bwd_dq_v10_kernel(const __grid_constant__ BwdMaps tm,
                                                                          AttnBwdProblem p) {
    constexpr int BMQ = 128, BKV = 128, CW = 2, KW = BKV / CW;
    using T = BT<HD>;
    constexpr int HDP = ((HD + 15) / 16) * 16;
    constexpr int S_COL = 0, DP_COL = 128, DS_COL = DP_COL + 32, DQ_COL = 256, Q_COL = 400;
    static_assert(DQ_COL + HDP <= Q_COL && Q_COL + HD / 2 <= 512, "TMEM budget");
    constexpr int KV_STAGE = 2 * T::T_TILE;  // two 64-key transposed tiles
    constexpr int NSV = 2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sdO = smem;
    uint8_t* sKt = sdO + T::ROW_TILE;    // [NS]
    uint8_t* sVt = sKt + NS * KV_STAGE;  // [NSV]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sVt + NSV * KV_STAGE);
    uint64_t* do_full = bars;
    uint64_t* kf = bars + 1;           // [NS]
    uint64_t* ke = kf + NS;            // [NS]
    uint64_t* vf = ke + NS;            // [NSV]
    uint64_t* ve = vf + NSV;           // [NSV]
    uint64_t* s_full = ve + NSV;
    uint64_t* s_empty = s_full + 1;
    uint64_t* dp_full = s_full + 2;
    uint64_t* ds_full = s_full + 3;
    uint64_t* acc_done = s_full + 4;
    uint64_t* qa_ready = s_full + 5;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 6);

    const AttnProblem& f = p.f;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int h = blockIdx.y, q0 = blockIdx.x * BMQ;
    // packed segments (AttnProblem::seg): this query tile's keys are its segment's
    const int klo = f.seg ? f.seg[2 * (q0 / 128)] : 0, khi = f.seg ? f.seg[2 * (q0 / 128) + 1] : f.Nk;
    const int nkv = (khi - klo + BKV - 1) / BKV;
    const int col = h * HD;

    if (threadIdx.x == 0) {
        mbar_init(do_full, 1);
        for (int i = 0; i < NS; ++i) {
            mbar_init(&kf[i], 1);
            mbar_init(&ke[i], 1);
        }
        for (int i = 0; i < NSV; ++i) {
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
                tma_load_2d(sKt + b * KV_STAGE, &tm.ta, &kf[b], klo + j * BKV, col);
                tma_load_2d(sKt + b * KV_STAGE + T::T_TILE, &tm.ta, &kf[b], klo + j * BKV + 64, col);
                const int bv = j % NSV;
                if (j >= NSV) mbar_wait(&ve[bv], ((j / NSV) - 1) & 1);
                mbar_arrive_expect_tx(&vf[bv], KV_STAGE);
                tma_load_2d(sVt + bv * KV_STAGE, &tm.tb, &vf[bv], klo + j * BKV, col);
                tma_load_2d(sVt + bv * KV_STAGE + T::T_TILE, &tm.tb, &vf[bv], klo + j * BKV + 64, col);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t id128 = idesc_bf16_f32(128, 128, false, true), idhd = idesc_bf16_f32(128, HD, false, false);
        auto issue_s = [&](int j) {  // S = Q K^T: A = Q from TMEM, B^T = the stage's HD x 128 K^T tiles (MN-major)
            const int b = j % NS;
            mbar_wait(&kf[b], (j / NS) & 1);
            if (j >= 1) mbar_wait(s_empty, (j - 1) & 1);
            tc_fence_after();
            if ((threadIdx.x & 31) == 0) ATR(0, j);
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
            const int b = j % NSV;
            mbar_wait(&vf[b], (j / NSV) & 1);
            tc_fence_after();
            if ((threadIdx.x & 31) == 0) ATR(2, j);
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
            if ((threadIdx.x & 31) == 0) ATR(1, j);
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
            if (warp == 4 && lane == 0) ATR(3, j);
            tmem_ld32(tmem + lane_base + S_COL + hf * KW, reinterpret_cast<uint32_t*>(pr));
            tmem_ld32(tmem + lane_base + S_COL + hf * KW + 32, reinterpret_cast<uint32_t*>(pr + 32));
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(s_empty);
            if (warp == 4 && lane == 0) ATR(4, j);
            const int kb = klo + j * BKV + hf * KW;
            if (kb + KW <= khi) {  // packed pairs: FFMA2 (bit-identical to the scalar fmaf)
                const float2 lg2 = make_float2(kLog2e, kLog2e), nl2 = make_float2(-lse2, -lse2);
#pragma unroll
                for (int c = 0; c < KW; c += 2) {
                    const float2 x = ffma2(make_float2(pr[c], pr[c + 1]), lg2, nl2);
                    if (MGV_DQ_X & 2) {
                        pr[c] = x.x;
                        pr[c + 1] = x.y;
                    } else {
                        pr[c] = ex2f(x.x);
                        pr[c + 1] = ex2f(x.y);
                    }
                }
            } else {
#pragma unroll
                for (int c = 0; c < KW; ++c) pr[c] = kb + c < khi ? ex2f(fmaf(pr[c], kLog2e, -lse2)) : 0.0f;
            }
            if (warp == 4 && lane == 0) ATR(5, j);
            mbar_wait(dp_full, j & 1);
            tc_fence_after();
            if (warp == 4 && lane == 0) ATR(6, j);
            float dp[KW];
            tmem_ld32(tmem + lane_base + DP_COL + hf * KW, reinterpret_cast<uint32_t*>(dp));
            tmem_ld32(tmem + lane_base + DP_COL + hf * KW + 32, reinterpret_cast<uint32_t*>(dp + 32));
            tmem_wait_ld();  // all of this warp's dP columns are in registers before its dS overwrites them
            uint32_t dk[KW / 2];
            const float2 D2 = make_float2(Dq, Dq);
#pragma unroll
            for (int c = 0; c < KW; c += 2) {  // dS = P (dP - D) (autodiff.cpp:820), packed pairs
                const float2 d = fmul2(make_float2(pr[c], pr[c + 1]), fsub2(make_float2(dp[c], dp[c + 1]), D2));
                dk[c / 2] = pack_bf16(d.x, d.y);
            }
            tmem_st16(tmem + lane_base + DS_COL + hf * (KW / 2), dk);
            tmem_st16(tmem + lane_base + DS_COL + hf * (KW / 2) + 16, dk + 16);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(ds_full);
            if (warp == 4 && lane == 0) ATR(7, j);
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
        const int smem = 2 * T::ROW_TILE + 4 * 2 * T::T_TILE + 4 * 128 * 4 + 256 + 1024;
        ensure_smem(attn_bwd_dkv_v11_kernel<HD, 2>, smem);
        // few key tiles (cross-attention): split the query range so the grid still covers the SMs
        const int kv_ctas = (f.Nk + 127) / 128 * f.heads, nq_all = (f.Nq + 127) / 128;
        const int splits = f.seg ? 1 : std::max(1, std::min({num_sms() / std::max(kv_ctas, 1), nq_all / 8, 16}));
        float* part = nullptr;
        if (splits > 1) MGV_CUDA(cudaMallocAsync(&part, sizeof(float) * splits * f.Nk * 2 * W, s));
        attn_bwd_dkv_v11_kernel<HD, 2><<<dim3((f.Nk + 127) / 128, f.heads, splits), 384, smem, s>>>(m, p, part);
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
        // Q rows are read straight into TMEM with 16-byte loads; dO row tiles by TMA
        if ((reinterpret_cast<uintptr_t>(f.q) | reinterpret_cast<uintptr_t>(p.dO)) % 16 || f.q_ld % 8 || p.do_ld % 8)
            throw std::runtime_error("attn_bwd_tc: q / dO must be 16-byte aligned with ld % 8 == 0");
        make_tmap_sw(&m.b128, p.dO, W, f.Nq, p.do_ld, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
        make_tmap_sw(&m.b32, p.dO, W, f.Nq, p.do_ld, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B);
        const int smem = T::ROW_TILE + (3 + 2) * 2 * T::T_TILE + 256 + 1024;
        ensure_smem(attn_bwd_dq_v10_kernel<HD, 3>, smem);
        attn_bwd_dq_v10_kernel<HD, 3><<<dim3((f.Nq + 127) / 128, f.heads), 128 + 128 * 2, smem, s>>>(m, p);
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
    const int64_t need = (static_cast<int64_t>(f.Nq) + 127) / 128 * 128;
    std::vector<float*> ftmp;
    if (lse_stride(f) < need || lse_stride(f) % 128 != 0) {
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

