// tcgen05 flash-attention backward for sm_100a, deterministic (no atomics):
// the gradient of Tape::mha (autodiff.cpp:795-843) computed in two passes.
//
//   dK/dV pass  CTA per (128-key tile, head), loops over 64-query tiles:
//                 S^T = K Q^T, dP^T = V dO^T            (TMEM, N = 64)
//                 P^T = exp(S^T - lse), dS^T = P^T (dP^T - D)   (thread = key row)
//                 dV += P^T dO, dK += dS^T Q            (TMEM accumulators, dO/Q read MN-major)
//   dQ pass     CTA per (128-query tile, head), loops over 64-key tiles:
//                 S = Q K^T, dP = dO V^T  (double-buffered in TMEM)
//                 dS = P (dP - D)                       (thread = query row)
//                 dQ += dS K                            (K read MN-major)
// The MMA warp software-pipelines the next tile's S/dP products under the
// current tile's elementwise work.  Layouts follow attn_tc.cu (64-col SW128
// chunks + 16-col SW32 tail for head_dim 144).
#include <cfloat>

#include "attn.h"
#include "gemm.cuh"
#include "ptx.cuh"

namespace mgv {

namespace {

constexpr float kLog2e = 1.4426950408889634f;

template <int HD, int R>
struct Tile {
    static constexpr int NF = HD / 64;
    static constexpr int TAIL = HD % 64;
    static constexpr int CH = R * 128;  // bytes of one 64-column SW128 chunk
    static constexpr int TB = R * 32;   // bytes of the 16-column SW32 tail
    static constexpr int BYTES = NF * CH + (TAIL ? TB : 0);
};

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int HD, int R>
__device__ __forceinline__ void load_tile_r(uint8_t* dst, const CUtensorMap* m128, const CUtensorMap* m32,
                                            uint64_t* bar, int col0, int row0) {
    using T = Tile<HD, R>;
#pragma unroll
    for (int c = 0; c < T::NF; ++c) tma_load_2d(dst + c * T::CH, m128, bar, col0 + c * 64, row0);
    if (T::TAIL) tma_load_2d(dst + T::NF * T::CH, m32, bar, col0 + T::NF * 64, row0);
}

// D (+)= A B^T with A (128 rows, K-major over HD) and B (N rows, K-major over HD).
template <int HD, int RA, int RB>
__device__ __forceinline__ void mma_kmajor_hd(uint32_t d, uint32_t a, uint32_t b, uint32_t idesc) {
    using TA = Tile<HD, RA>;
    using TB = Tile<HD, RB>;
    int kk = 0;
#pragma unroll
    for (int c = 0; c < TA::NF; ++c)
#pragma unroll
        for (int k = 0; k < 4; ++k, ++kk)
            umma_f16_ss(d, smem_desc(a + c * TA::CH + k * 32, 16, 1024, kSwizzle128),
                        smem_desc(b + c * TB::CH + k * 32, 16, 1024, kSwizzle128), idesc, kk > 0);
    if (TA::TAIL)
        umma_f16_ss(d, smem_desc(a + TA::NF * TA::CH, 16, 256, kSwizzle32),
                    smem_desc(b + TB::NF * TB::CH, 16, 256, kSwizzle32), idesc, 1);
}

// D[128 x HD] (+)= A[128 x KR] * B where A is a 128 x KR bf16 K-major SW128 chunk (KR = 64)
// and B is an R=KR-row tile [KR][HD] read MN-major (N = HD split 128|64 + 16).
template <int HD, int KR>
__device__ __forceinline__ void mma_mn_hd(uint32_t d, uint32_t a, uint32_t b, bool acc_first) {
    using TB = Tile<HD, KR>;
    constexpr uint32_t idA = idesc_bf16_f32(128, TB::NF >= 2 ? 128 : 64, false, true);
    constexpr uint32_t idT = idesc_bf16_f32(128, 16, false, true);
#pragma unroll
    for (int ks = 0; ks < KR / 16; ++ks) {
        const uint64_t ad = smem_desc(a + ks * 32, 16, 1024, kSwizzle128);
        const uint32_t acc = (acc_first || ks > 0) ? 1u : 0u;
        umma_f16_ss(d, ad, smem_desc(b + ks * 2048, TB::CH, 1024, kSwizzle128), idA, acc);
        if (TB::TAIL) umma_f16_ss(d + TB::NF * 64, ad, smem_desc(b + TB::NF * TB::CH + ks * 512, 0, 256, kSwizzle32), idT, acc);
    }
}

// Row (thread) -> 64 bf16 values into a 128 x 64 SW128 K-major chunk.
__device__ __forceinline__ void st_row64(uint8_t* chunk, int row, const uint32_t* pk) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
        *reinterpret_cast<uint4*>(chunk + row * 128 + ((u ^ (row & 7)) << 4)) =
            make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
}

template <int HD>
__device__ __forceinline__ void store_acc_row(uint32_t taddr, __nv_bfloat16* out, bool valid) {
#pragma unroll 1
    for (int c = 0; c < HD / 16; ++c) {
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

struct BwdMaps {
    CUtensorMap k128, k32, v128, v32;    // key tiles
    CUtensorMap q128, q32, do128, do32;  // query tiles
};

}  // namespace

// =====================================================================================  dK / dV
template <int HD>
__global__ void __launch_bounds__(256, 1) attn_bwd_dkv_tc_kernel(const __grid_constant__ BwdMaps tm, AttnBwdProblem p) {
    constexpr int BKV = 128, BQ = 64;
    using TK = Tile<HD, BKV>;
    using TQ = Tile<HD, BQ>;
    constexpr int DV_COL = 128, DK_COL = HD <= 128 ? 256 : 320;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sK = smem;
    uint8_t* sV = sK + TK::BYTES;
    uint8_t* sQ = sV + TK::BYTES;          // [2]
    uint8_t* sdO = sQ + 2 * TQ::BYTES;     // [2]
    uint8_t* sPT = sdO + 2 * TQ::BYTES;    // [2] x 16 KB
    uint8_t* sdST = sPT + 2 * 16384;       // [2] x 16 KB
    float* sLse = reinterpret_cast<float*>(sdST + 2 * 16384);  // [2][64] (log2 domain)
    float* sD = sLse + 2 * BQ;                                  // [2][64]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sD + 2 * BQ);
    uint64_t* kv_full = bars;
    uint64_t* qd_full = bars + 1;   // [2]
    uint64_t* qd_empty = bars + 3;  // [2]
    uint64_t* lse_full = bars + 5;  // [2]
    uint64_t* s_full = bars + 7;
    uint64_t* s_empty = bars + 8;
    uint64_t* p_full = bars + 9;
    uint64_t* pd_done = bars + 10;  // [2]
    uint64_t* acc_done = bars + 12;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

    const AttnProblem& f = p.f;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int h = blockIdx.y, k0 = blockIdx.x * BKV;
    const int nq = (f.Nq + BQ - 1) / BQ;
    const int col = h * HD;

    if (threadIdx.x == 0) {
        mbar_init(kv_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&qd_full[i], 1);
            mbar_init(&qd_empty[i], 1);
            mbar_init(&lse_full[i], 32);
            mbar_init(&pd_done[i], 1);
        }
        mbar_init(s_full, 1);
        mbar_init(s_empty, 4);
        mbar_init(p_full, 4);
        mbar_init(acc_done, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- producer: K, V once; Q, dO, lse, D per query tile
        if (lane == 0) {
            mbar_arrive_expect_tx(kv_full, 2 * TK::BYTES);
            load_tile_r<HD, BKV>(sK, &tm.k128, &tm.k32, kv_full, col, k0);
            load_tile_r<HD, BKV>(sV, &tm.v128, &tm.v32, kv_full, col, k0);
        }
        for (int i = 0; i < nq; ++i) {
            const int st = i & 1;
            if (i >= 2) mbar_wait(&qd_empty[st], ((i - 2) >> 1) & 1);
            if (lane == 0) {
                mbar_arrive_expect_tx(&qd_full[st], 2 * TQ::BYTES);
                load_tile_r<HD, BQ>(sQ + st * TQ::BYTES, &tm.q128, &tm.q32, &qd_full[st], col, i * BQ);
                load_tile_r<HD, BQ>(sdO + st * TQ::BYTES, &tm.do128, &tm.do32, &qd_full[st], col, i * BQ);
            }
            for (int c = lane; c < BQ; c += 32) {
                const int q = i * BQ + c;
                sLse[st * BQ + c] = q < f.Nq ? f.lse[(int64_t)h * f.Nq + q] * kLog2e : 0.0f;
                sD[st * BQ + c] = q < f.Nq ? p.Dvec[(int64_t)h * f.Nq + q] : 0.0f;
            }
            mbar_arrive(&lse_full[st]);
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        constexpr uint32_t idS = idesc_bf16_f32(128, BQ, false, false);
        const uint32_t aK = smem_u32(sK), aV = smem_u32(sV);
        auto issue_s = [&](int i) {
            const int st = i & 1;
            mma_kmajor_hd<HD, BKV, BQ>(tmem + 0, aK, smem_u32(sQ + st * TQ::BYTES), idS);
            mma_kmajor_hd<HD, BKV, BQ>(tmem + 64, aV, smem_u32(sdO + st * TQ::BYTES), idS);
        };
        mbar_wait(kv_full, 0);
        if (nq > 0) {
            mbar_wait(&qd_full[0], 0);
            tc_fence_after();
            if (elect_one()) {
                issue_s(0);
                umma_commit(s_full);
            }
            __syncwarp();
        }
        for (int i = 0; i < nq; ++i) {
            const int st = i & 1;
            if (i + 1 < nq) {
                mbar_wait(&qd_full[(i + 1) & 1], ((i + 1) >> 1) & 1);
                mbar_wait(s_empty, i & 1);  // softmax(i) has read S^T_i / dP^T_i
                tc_fence_after();
                if (elect_one()) {
                    issue_s(i + 1);
                    umma_commit(s_full);
                }
                __syncwarp();
            }
            mbar_wait(p_full, i & 1);
            tc_fence_after();
            if (elect_one()) {
                mma_mn_hd<HD, BQ>(tmem + DV_COL, smem_u32(sPT + st * 16384), smem_u32(sdO + st * TQ::BYTES), i > 0);
                mma_mn_hd<HD, BQ>(tmem + DK_COL, smem_u32(sdST + st * 16384), smem_u32(sQ + st * TQ::BYTES), i > 0);
                umma_commit(&pd_done[st]);
                umma_commit(&qd_empty[st]);
                if (i == nq - 1) umma_commit(acc_done);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ---------------- elementwise: thread = key row
        const int wq = warp - 4, row = wq * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
        for (int i = 0; i < nq; ++i) {
            const int st = i & 1;
            mbar_wait(&lse_full[st], (i >> 1) & 1);
            mbar_wait(s_full, i & 1);
            tc_fence_after();
            float s[BQ], dp[BQ];
            tmem_ld32(tmem + lane_base + 0, reinterpret_cast<uint32_t*>(s));
            tmem_ld32(tmem + lane_base + 32, reinterpret_cast<uint32_t*>(s + 32));
            tmem_ld32(tmem + lane_base + 64, reinterpret_cast<uint32_t*>(dp));
            tmem_ld32(tmem + lane_base + 96, reinterpret_cast<uint32_t*>(dp + 32));
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(s_empty);
            const float* lse2 = sLse + st * BQ;
            const float* Dq = sD + st * BQ;
            uint32_t pk[BQ / 2], dk[BQ / 2];
#pragma unroll
            for (int c = 0; c < BQ; c += 2) {
                const bool v0 = i * BQ + c < f.Nq, v1 = i * BQ + c + 1 < f.Nq;
                const float p0 = v0 ? ex2f(fmaf(s[c], kLog2e, -lse2[c])) : 0.0f;
                const float p1 = v1 ? ex2f(fmaf(s[c + 1], kLog2e, -lse2[c + 1])) : 0.0f;
                pk[c / 2] = pack_bf16(p0, p1);
                dk[c / 2] = pack_bf16(p0 * (dp[c] - Dq[c]), p1 * (dp[c + 1] - Dq[c + 1]));  // autodiff.cpp:820
            }
            if (i >= 2) mbar_wait(&pd_done[st], ((i - 2) >> 1) & 1);
            st_row64(sPT + st * 16384, row, pk);
            st_row64(sdST + st * 16384, row, dk);
            fence_proxy_async();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(p_full);
        }
        if (nq > 0) mbar_wait(acc_done, 0);
        tc_fence_after();
        const int kv = k0 + row;
        const bool valid = kv < f.Nk && nq > 0;
        store_acc_row<HD>(tmem + lane_base + DV_COL, static_cast<__nv_bfloat16*>(p.dv) + (int64_t)kv * p.dv_ld + col,
                          valid);
        store_acc_row<HD>(tmem + lane_base + DK_COL, static_cast<__nv_bfloat16*>(p.dk) + (int64_t)kv * p.dk_ld + col,
                          valid);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

// =====================================================================================  dQ
template <int HD>
__global__ void __launch_bounds__(256, 1) attn_bwd_dq_tc_kernel(const __grid_constant__ BwdMaps tm, AttnBwdProblem p) {
    constexpr int BMQ = 128, BKV = 64;
    using TQ = Tile<HD, BMQ>;
    using TK = Tile<HD, BKV>;
    constexpr int DQ_COL = 256;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sdO = sQ + TQ::BYTES;
    uint8_t* sK = sdO + TQ::BYTES;    // [2]
    uint8_t* sV = sK + 2 * TK::BYTES;  // [2]
    uint8_t* sdS = sV + 2 * TK::BYTES;  // [2] x 16 KB
    uint64_t* bars = reinterpret_cast<uint64_t*>(sdS + 2 * 16384);
    uint64_t* q_full = bars;
    uint64_t* kv_full = bars + 1;   // [2]
    uint64_t* kv_empty = bars + 3;  // [2]
    uint64_t* s_full = bars + 5;    // [2]
    uint64_t* s_empty = bars + 7;   // [2]
    uint64_t* ds_full = bars + 9;
    uint64_t* ds_empty = bars + 10;  // [2]
    uint64_t* acc_done = bars + 12;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

    const AttnProblem& f = p.f;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int h = blockIdx.y, q0 = blockIdx.x * BMQ;
    const int nkv = (f.Nk + BKV - 1) / BKV;
    const int col = h * HD;

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&s_empty[i], 4);
            mbar_init(&ds_empty[i], 1);
        }
        mbar_init(ds_full, 4);
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
            mbar_arrive_expect_tx(q_full, 2 * TQ::BYTES);
            load_tile_r<HD, BMQ>(sQ, &tm.q128, &tm.q32, q_full, col, q0);
            load_tile_r<HD, BMQ>(sdO, &tm.do128, &tm.do32, q_full, col, q0);
            for (int j = 0; j < nkv; ++j) {
                const int b = j & 1;
                if (j >= 2) mbar_wait(&kv_empty[b], ((j - 2) >> 1) & 1);
                mbar_arrive_expect_tx(&kv_full[b], 2 * TK::BYTES);
                load_tile_r<HD, BKV>(sK + b * TK::BYTES, &tm.k128, &tm.k32, &kv_full[b], col, j * BKV);
                load_tile_r<HD, BKV>(sV + b * TK::BYTES, &tm.v128, &tm.v32, &kv_full[b], col, j * BKV);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idS = idesc_bf16_f32(128, BKV, false, false);
        const uint32_t aQ = smem_u32(sQ), adO = smem_u32(sdO);
        auto issue_dq = [&](int j) {
            const int b = j & 1;
            mma_mn_hd<HD, BKV>(tmem + DQ_COL, smem_u32(sdS + b * 16384), smem_u32(sK + b * TK::BYTES), j > 0);
            umma_commit(&ds_empty[b]);
            umma_commit(&kv_empty[b]);
        };
        mbar_wait(q_full, 0);
        for (int j = 0; j < nkv; ++j) {
            const int b = j & 1;
            mbar_wait(&kv_full[b], (j >> 1) & 1);
            if (j >= 2) mbar_wait(&s_empty[b], ((j - 2) >> 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                mma_kmajor_hd<HD, BMQ, BKV>(tmem + b * 128, aQ, smem_u32(sK + b * TK::BYTES), idS);
                mma_kmajor_hd<HD, BMQ, BKV>(tmem + b * 128 + 64, adO, smem_u32(sV + b * TK::BYTES), idS);
                umma_commit(&s_full[b]);
            }
            __syncwarp();
            if (j >= 1) {
                mbar_wait(ds_full, (j - 1) & 1);
                tc_fence_after();
                if (elect_one()) issue_dq(j - 1);
                __syncwarp();
            }
        }
        if (nkv > 0) {
            mbar_wait(ds_full, (nkv - 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                issue_dq(nkv - 1);
                umma_commit(acc_done);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        const int wq = warp - 4, row = wq * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
        const int q = q0 + row;
        const float lse2 = q < f.Nq ? f.lse[(int64_t)h * f.Nq + q] * kLog2e : 0.0f;
        const float Dq = q < f.Nq ? p.Dvec[(int64_t)h * f.Nq + q] : 0.0f;
        for (int j = 0; j < nkv; ++j) {
            const int b = j & 1;
            mbar_wait(&s_full[b], (j >> 1) & 1);
            tc_fence_after();
            float s[BKV], dp[BKV];
            tmem_ld32(tmem + lane_base + b * 128, reinterpret_cast<uint32_t*>(s));
            tmem_ld32(tmem + lane_base + b * 128 + 32, reinterpret_cast<uint32_t*>(s + 32));
            tmem_ld32(tmem + lane_base + b * 128 + 64, reinterpret_cast<uint32_t*>(dp));
            tmem_ld32(tmem + lane_base + b * 128 + 96, reinterpret_cast<uint32_t*>(dp + 32));
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[b]);
            uint32_t dk[BKV / 2];
#pragma unroll
            for (int c = 0; c < BKV; c += 2) {
                const bool v0 = j * BKV + c < f.Nk, v1 = j * BKV + c + 1 < f.Nk;
                const float p0 = v0 ? ex2f(fmaf(s[c], kLog2e, -lse2)) : 0.0f;
                const float p1 = v1 ? ex2f(fmaf(s[c + 1], kLog2e, -lse2)) : 0.0f;
                dk[c / 2] = pack_bf16(p0 * (dp[c] - Dq), p1 * (dp[c + 1] - Dq));
            }
            if (j >= 2) mbar_wait(&ds_empty[b], ((j - 2) >> 1) & 1);
            st_row64(sdS + b * 16384, row, dk);
            fence_proxy_async();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(ds_full);
        }
        if (nkv > 0) mbar_wait(acc_done, 0);
        tc_fence_after();
        store_acc_row<HD>(tmem + lane_base + DQ_COL, static_cast<__nv_bfloat16*>(p.dq) + (int64_t)q * p.dq_ld + col,
                          q < f.Nq && nkv > 0);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ host
template <int HD>
static void make_maps(BwdMaps* m, const AttnBwdProblem& p, int krows, int qrows) {
    const AttnProblem& f = p.f;
    const uint64_t W = (uint64_t)f.heads * HD;
    make_tmap_sw(&m->k128, f.k, W, f.Nk, f.k_ld, 64, krows, CU_TENSOR_MAP_SWIZZLE_128B);
    make_tmap_sw(&m->k32, f.k, W, f.Nk, f.k_ld, 16, krows, CU_TENSOR_MAP_SWIZZLE_32B);
    make_tmap_sw(&m->v128, f.v, W, f.Nk, f.v_ld, 64, krows, CU_TENSOR_MAP_SWIZZLE_128B);
    make_tmap_sw(&m->v32, f.v, W, f.Nk, f.v_ld, 16, krows, CU_TENSOR_MAP_SWIZZLE_32B);
    make_tmap_sw(&m->q128, f.q, W, f.Nq, f.q_ld, 64, qrows, CU_TENSOR_MAP_SWIZZLE_128B);
    make_tmap_sw(&m->q32, f.q, W, f.Nq, f.q_ld, 16, qrows, CU_TENSOR_MAP_SWIZZLE_32B);
    make_tmap_sw(&m->do128, p.dO, W, f.Nq, p.do_ld, 64, qrows, CU_TENSOR_MAP_SWIZZLE_128B);
    make_tmap_sw(&m->do32, p.dO, W, f.Nq, p.do_ld, 16, qrows, CU_TENSOR_MAP_SWIZZLE_32B);
}

template <int HD>
static void launch_bwd(const AttnBwdProblem& p, cudaStream_t s) {
    attn_bwd_dvec(p, s);
    {
        using TK = Tile<HD, 128>;
        using TQ = Tile<HD, 64>;
        const int smem = 2 * TK::BYTES + 4 * TQ::BYTES + 4 * 16384 + 4 * 64 * 4 + 256 + 1024;
        BwdMaps m;
        make_maps<HD>(&m, p, 128, 64);
        static bool set = false;
        if (!set) {
            MGV_CUDA(cudaFuncSetAttribute(attn_bwd_dkv_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            set = true;
        }
        attn_bwd_dkv_tc_kernel<HD><<<dim3((p.f.Nk + 127) / 128, p.f.heads), 256, smem, s>>>(m, p); ::mgv::note_launch();
        MGV_CUDA(cudaGetLastError());
    }
    {
        using TQ = Tile<HD, 128>;
        using TK = Tile<HD, 64>;
        const int smem = 2 * TQ::BYTES + 4 * TK::BYTES + 2 * 16384 + 256 + 1024;
        BwdMaps m;
        make_maps<HD>(&m, p, 64, 128);
        static bool set = false;
        if (!set) {
            MGV_CUDA(cudaFuncSetAttribute(attn_bwd_dq_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            set = true;
        }
        attn_bwd_dq_tc_kernel<HD><<<dim3((p.f.Nq + 127) / 128, p.f.heads), 256, smem, s>>>(m, p); ::mgv::note_launch();
        MGV_CUDA(cudaGetLastError());
    }
}

void attn_bwd_tc(const AttnBwdProblem& p, cudaStream_t s) {
    switch (p.f.hd) {
        case 64: launch_bwd<64>(p, s); break;
        case 128: launch_bwd<128>(p, s); break;
        case 144: launch_bwd<144>(p, s); break;
        default: throw std::runtime_error("attn_bwd_tc: unsupported head_dim");
    }
}

}  // namespace mgv
