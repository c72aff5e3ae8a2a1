// tcgen05 flash attention forward for sm_100a (bf16 operands, fp32 softmax and
// accumulation) -- Tape::mha forward (autodiff.cpp:755-793) at head_dim 144.
//
// One CTA per (256 queries = two 128-row tiles A and B, head), 12 warps:
//   warp 0        TMA producer: Q_A, Q_B once; then 112-key K tiles and V^T tiles
//                 through a 2-stage ring (each K/V byte now serves 256 queries)
//   warp 1        MMA issuer, ping-pong between the tiles:
//                   S_A(j), PV_B(j-1), S_B(j), PV_A(j), S_A(j+1), ...
//                 so the tensor core works on one tile while the other tile's
//                 softmax runs.  P is read straight from TMEM (TS form).
//   warp 2        TMEM allocator: S/P_A [0,112) S/P_B [112,224) O_A [224,368) O_B [368,512)
//   warps 4..7    softmax of tile A  } thread i = query row i = TMEM lane i:
//   warps 8..11   softmax of tile B  } tcgen05.ld S -> online softmax (log2 domain,
//                 ex2.approx) -> bf16 P over S (tcgen05.st) -> signal.  O is rescaled
//                 in TMEM only when the running max grows by more than 2^8.
// Registers are rebalanced with setmaxnreg (producer group 56, softmax groups 224).
//
// head_dim 144 = 64 + 64 + 16: Q and K tiles are 64-column SW128 chunks plus a
// 16-column SW32 tail (S = Q K^T = 9 K-steps, N = 112); V is consumed transposed
// (V^T tile = 144 rows x 128 keys, K-major) so O += P V is one N = 144 MMA per
// 16-key step (7 steps per 112-key tile).
#include <cfloat>
#include <cstdlib>

#include "attn.h"
#include "gemm.cuh"
#include "kernels.h"
#include "ptx.cuh"

namespace mgv {

namespace {

constexpr int BM = 128;  // queries per tile (two tiles per CTA)
constexpr int BN = 112;  // keys per step (TMEM: 2 x (112 + 144) = 512 columns)
constexpr float kLog2e = 1.4426950408889634f;

template <int HD>
struct FwdCfg {
    static constexpr int NF = HD / 64;
    static constexpr int TAIL = HD % 64;
    static_assert(TAIL == 0 || TAIL == 16, "head_dim must be 64k or 64k+16");
    static constexpr int Q_TILE = NF * 16384 + (TAIL ? 4096 : 0);    // 128 rows x HD
    static constexpr int K_CHUNK = BN * 128;                          // 112 rows x 64 cols (SW128)
    static constexpr int K_BYTES = NF * K_CHUNK + (TAIL ? BN * 32 : 0);  // TMA transaction bytes
    static constexpr int K_TILE = (K_BYTES + 1023) / 1024 * 1024;        // smem footprint (1 KB aligned)
    static constexpr int VT_CHUNK = HD * 128;                         // HD rows x 64 keys (SW128)
    static constexpr int VT_TILE = 2 * VT_CHUNK;                      // HD rows x 128 keys (112 used)
    static constexpr int STAGE = K_TILE + VT_TILE;
    static constexpr int SMEM = 2 * Q_TILE + 2 * STAGE + 1024 + 256;
    __host__ __device__ static constexpr int s_col(int t) { return t * BN; }
    __host__ __device__ static constexpr int o_col(int t) { return 2 * BN + t * HD; }
    static_assert(2 * BN + 2 * HD <= 512, "TMEM budget");
};

struct FwdMaps {
    CUtensorMap q128, q32, k128, k32, vt;
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int HD, int ROWS>
__device__ __forceinline__ void load_rows(uint8_t* dst, const CUtensorMap* m128, const CUtensorMap* m32,
                                          uint64_t* bar, int col0, int row0) {
    using C = FwdCfg<HD>;
#pragma unroll
    for (int c = 0; c < C::NF; ++c) tma_load_2d(dst + c * ROWS * 128, m128, bar, col0 + c * 64, row0);
    if (C::TAIL) tma_load_2d(dst + C::NF * ROWS * 128, m32, bar, col0 + C::NF * 64, row0);
}

}  // namespace

template <int HD>
__global__ void __launch_bounds__(384, 1) attn_fwd_tc_kernel(const __grid_constant__ FwdMaps tm, AttnProblem p) {
    using C = FwdCfg<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                      // [2] tiles
    uint8_t* sStage = sQ + 2 * C::Q_TILE;    // [2] x (K tile | V^T tile)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + 2 * C::STAGE);
    uint64_t* q_full = bars;         // both Q tiles
    uint64_t* k_full = bars + 1;     // [2]
    uint64_t* v_full = bars + 3;     // [2]
    uint64_t* kv_empty = bars + 5;   // [2]
    uint64_t* s_full = bars + 7;     // [tile]
    uint64_t* p_full = bars + 9;     // [tile]
    uint64_t* pv_done = bars + 11;   // [tile]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int h = blockIdx.y, q0 = blockIdx.x * 2 * BM;
    // packed segments (AttnProblem::seg): this CTA's 256 queries lie in one segment; its keys are that segment's
    const int klo = p.seg ? p.seg[2 * (q0 / 128)] : 0, khi = p.seg ? p.seg[2 * (q0 / 128) + 1] : p.Nk;
    const int nkv = (khi - klo + BN - 1) / BN;
    const int col = h * HD;

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&kv_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 4);
            mbar_init(&pv_done[i], 1);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 4) {
        setmaxnreg_dec<56>();
        if (warp == 0) {
            if (elect_one()) {
                tma_prefetch(&tm.q128);
                tma_prefetch(&tm.k128);
                tma_prefetch(&tm.vt);
                mbar_arrive_expect_tx(q_full, 2 * C::Q_TILE);
                load_rows<HD, BM>(sQ, &tm.q128, &tm.q32, q_full, col, q0);
                load_rows<HD, BM>(sQ + C::Q_TILE, &tm.q128, &tm.q32, q_full, col, q0 + BM);
                for (int j = 0; j < nkv; ++j) {
                    const int st = j & 1;
                    if (j >= 2) mbar_wait(&kv_empty[st], ((j - 2) >> 1) & 1);
                    uint8_t* sK = sStage + st * C::STAGE;
                    uint8_t* sVt = sK + C::K_TILE;
                    mbar_arrive_expect_tx(&k_full[st], C::K_BYTES);
                    load_rows<HD, BN>(sK, &tm.k128, &tm.k32, &k_full[st], col, klo + j * BN);
                    mbar_arrive_expect_tx(&v_full[st], C::VT_TILE);
                    tma_load_2d(sVt, &tm.vt, &v_full[st], klo + j * BN, col);
                    tma_load_2d(sVt + C::VT_CHUNK, &tm.vt, &v_full[st], klo + j * BN + 64, col);
                }
            }
        } else if (warp == 1) {
            constexpr uint32_t idS = idesc_bf16_f32(BM, BN, false, false);
            constexpr uint32_t idO = idesc_bf16_f32(BM, HD, false, false);
            auto issue_s = [&](int t, int j) {
                const uint32_t aQ = smem_u32(sQ + t * C::Q_TILE);
                const uint32_t aK = smem_u32(sStage + (j & 1) * C::STAGE);
                const uint32_t d = tmem + C::s_col(t);
                int kk = 0;
#pragma unroll
                for (int c = 0; c < C::NF; ++c)
#pragma unroll
                    for (int k = 0; k < 4; ++k, ++kk)
                        umma_f16_ss(d, smem_desc(aQ + c * 16384 + k * 32, 16, 1024, kSwizzle128),
                                    smem_desc(aK + c * C::K_CHUNK + k * 32, 16, 1024, kSwizzle128), idS, kk > 0);
                if (C::TAIL)
                    umma_f16_ss(d, smem_desc(aQ + C::NF * 16384, 16, 256, kSwizzle32),
                                smem_desc(aK + C::NF * C::K_CHUNK, 16, 256, kSwizzle32), idS, 1);
                umma_commit(&s_full[t]);
            };
            auto issue_pv = [&](int t, int j) {
                const uint32_t aVt = smem_u32(sStage + (j & 1) * C::STAGE + C::K_TILE);
                const uint32_t pt = tmem + C::s_col(t);  // bf16 P packed 2 per column over S
#pragma unroll
                for (int ks = 0; ks < BN / 16; ++ks)
                    umma_f16_ts(tmem + C::o_col(t), pt + ks * 8,
                                smem_desc(aVt + (ks >> 2) * C::VT_CHUNK + (ks & 3) * 32, 16, 1024, kSwizzle128), idO,
                                (j > 0 || ks > 0) ? 1u : 0u);
                umma_commit(&pv_done[t]);
            };
            mbar_wait(q_full, 0);
            for (int j = 0; j <= nkv; ++j) {
                if (j < nkv) {
                    mbar_wait(&k_full[j & 1], (j >> 1) & 1);
                    tc_fence_after();
                    if (elect_one()) issue_s(0, j);  // S_A(j): P_A(j-1) consumed by PV_A(j-1), issued earlier
                    __syncwarp();
                }
                if (j >= 1) {  // PV_B(j-1), then the stage of step j-1 is free
                    mbar_wait(&p_full[1], (j - 1) & 1);
                    tc_fence_after();
                    if (elect_one()) {
                        issue_pv(1, j - 1);
                        umma_commit(&kv_empty[(j - 1) & 1]);
                    }
                    __syncwarp();
                }
                if (j < nkv) {
                    if (elect_one()) issue_s(1, j);  // S_B(j)
                    __syncwarp();
                    mbar_wait(&p_full[0], j & 1);
                    mbar_wait(&v_full[j & 1], (j >> 1) & 1);
                    tc_fence_after();
                    if (elect_one()) issue_pv(0, j);  // PV_A(j)
                    __syncwarp();
                }
            }
        }
    } else {
        // ------------------------------------------------ softmax, tile t = 0 (warps 4-7) or 1 (8-11)
        setmaxnreg_inc<224>();
        const int t = (warp - 4) >> 2, wq = warp & 3;
        const int row = wq * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
        const uint32_t sS = tmem + lane_base + C::s_col(t);
        const uint32_t sO = tmem + lane_base + C::o_col(t);
        float m2 = -FLT_MAX;  // running max (log2 domain)
        float l = 0.0f;
        for (int j = 0; j < nkv; ++j) {
            mbar_wait(&s_full[t], j & 1);
            tc_fence_after();
            float s[BN];
            tmem_ld32(sS + 0, reinterpret_cast<uint32_t*>(s));
            tmem_ld32(sS + 32, reinterpret_cast<uint32_t*>(s + 32));
            tmem_ld32(sS + 64, reinterpret_cast<uint32_t*>(s + 64));
            tmem_ld16(sS + 96, reinterpret_cast<uint32_t*>(s + 96));
            tmem_wait_ld();
            const int kv0 = klo + j * BN;
            if (kv0 + BN > khi) {
#pragma unroll
                for (int c = 0; c < BN; ++c)
                    if (kv0 + c >= khi) s[c] = -FLT_MAX;
            }
            float mx8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) mx8[e] = s[e];
#pragma unroll
            for (int c = 8; c < BN; c += 8)
#pragma unroll
                for (int e = 0; e < 8; ++e) mx8[e] = fmaxf(mx8[e], s[c + e]);
            const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                   fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * kLog2e;
            float alpha = 1.0f, m_use = m2;
            if (j == 0) {
                m_use = mx;
            } else if (mx > m2 + 8.0f) {
                m_use = mx;
                alpha = ex2(m2 - mx);
            }
            // the softmax warps are issue-bound: the scale/shift and the row sum run as packed f32x2
            // instructions (FFMA2 / FADD2), two columns per instruction
            float2 ps2[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) ps2[e] = make_float2(0.0f, 0.0f);
            const float2 lg2 = make_float2(kLog2e, kLog2e), nm2 = make_float2(-m_use, -m_use);
            uint32_t pk[BN / 2];
#pragma unroll
            for (int c = 0; c < BN; c += 2) {
                const float2 x = ffma2(make_float2(s[c], s[c + 1]), lg2, nm2);
                float2 pp;
                pp.x = ex2(x.x);
                pp.y = ex2(x.y);
                ps2[(c / 2) & 3] = fadd2(ps2[(c / 2) & 3], pp);
                pk[c / 2] = pack_bf16(pp.x, pp.y);
            }
            const float ps = ((ps2[0].x + ps2[0].y) + (ps2[1].x + ps2[1].y)) + ((ps2[2].x + ps2[2].y) + (ps2[3].x + ps2[3].y));
            if (j >= 1 && __any_sync(0xffffffff, alpha != 1.0f)) {
                mbar_wait(&pv_done[t], (j - 1) & 1);  // O holds exactly PV(0..j-1)
                tc_fence_after();
#pragma unroll 1
                for (int c = 0; c < HD / 16; ++c) {
                    uint32_t r[16];
                    tmem_ld16(sO + c * 16, r);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 16; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
                    tmem_st16(sO + c * 16, r);
                }
            }
            l = l * alpha + ps;
            m2 = m_use;
            tmem_st32(sS + 0, pk);  // 56 packed columns over S
            tmem_st16(sS + 32, pk + 32);
            tmem_st8(sS + 48, pk + 48);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[t]);
        }
        if (nkv > 0) {
            mbar_wait(&pv_done[t], (nkv - 1) & 1);
            tc_fence_after();
        }
        const int q = q0 + t * BM + row;
        const float inv = l > 0.0f ? 1.0f / l : 0.0f;
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.o) + (int64_t)q * p.o_ld + col;
#pragma unroll 1
        for (int c = 0; c < HD / 16; ++c) {
            uint32_t r[16];
            tmem_ld16(sO + c * 16, r);
            tmem_wait_ld();
            if (q < p.Nq) {
                uint32_t o[8];
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    o[e] = pack_bf16(__uint_as_float(r[2 * e]) * inv, __uint_as_float(r[2 * e + 1]) * inv);
                uint4* dst = reinterpret_cast<uint4*>(out + c * 16);
                dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
                dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
            }
        }
        if (q < p.Nq) p.lse[(int64_t)h * lse_stride(p) + q] = (m2 + __log2f(l)) * 0.6931471805599453f;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ host
bool attn_tc_supported(int hd, int Nk) {
    (void)Nk;
    return hd == 64 || hd == 128 || hd == 144;
}

template <int HD>
static void launch_fwd(const AttnProblem& p, const void* vt, int64_t vt_ld, cudaStream_t s) {
    using C = FwdCfg<HD>;
    FwdMaps tm;
    const uint64_t W = (uint64_t)p.heads * HD;
    make_tmap_sw(&tm.q128, p.q, W, p.Nq, p.q_ld, 64, BM, CU_TENSOR_MAP_SWIZZLE_128B);
    make_tmap_sw(&tm.q32, p.q, W, p.Nq, p.q_ld, 16, BM, CU_TENSOR_MAP_SWIZZLE_32B);
    make_tmap_sw(&tm.k128, p.k, W, p.Nk, p.k_ld, 64, BN, CU_TENSOR_MAP_SWIZZLE_128B);
    make_tmap_sw(&tm.k32, p.k, W, p.Nk, p.k_ld, 16, BN, CU_TENSOR_MAP_SWIZZLE_32B);
    // V^T: rows = heads*HD (dims), cols = keys; box = 64 keys x HD dims
    make_tmap_sw(&tm.vt, vt, p.Nk, W, vt_ld, 64, HD, CU_TENSOR_MAP_SWIZZLE_128B);
    ensure_smem(attn_fwd_tc_kernel<HD>, C::SMEM);
    dim3 grid((p.Nq + 2 * BM - 1) / (2 * BM), p.heads);
    attn_fwd_tc_kernel<HD><<<grid, 384, C::SMEM, s>>>(tm, p);
    ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

void attn_fwd_tc(const AttnProblem& p, cudaStream_t s) {
    const void* vt = p.vt;
    int64_t vt_ld = p.vt_ld;
    __nv_bfloat16* tmp = nullptr;
    if (!vt) {  // transpose V here (callers that keep V^T for the backward pass supply it)
        vt_ld = (p.Nk + 7) / 8 * 8;
        MGV_CUDA(cudaMallocAsync(&tmp, sizeof(__nv_bfloat16) * vt_ld * p.heads * p.hd, s));
        transpose_bf16(static_cast<const __nv_bfloat16*>(p.v), p.v_ld, p.Nk, p.heads * p.hd, tmp, vt_ld, s);
        vt = tmp;
    }
    switch (p.hd) {
        case 64: launch_fwd<64>(p, vt, vt_ld, s); break;
        case 128: launch_fwd<128>(p, vt, vt_ld, s); break;
        case 144: launch_fwd<144>(p, vt, vt_ld, s); break;
        default: throw std::runtime_error("attn_fwd_tc: unsupported head_dim");
    }
    if (tmp) MGV_CUDA(cudaFreeAsync(tmp, s));
}

}  // namespace mgv

extern "C" {
// Op-level entry for tests / roofline: bf16 operands, token-major with row strides; tc != 0 selects tcgen05.
int mgv_dev_attn_fwd(int tc, const void* q, int64_t q_ld, const void* k, int64_t k_ld, const void* v, int64_t v_ld,
                     void* o, int64_t o_ld, float* lse, int Nq, int Nk, int heads, int hd, void* stream) {
    try {
        mgv::AttnProblem p{q, q_ld, k, k_ld, v, v_ld, o, o_ld, lse, Nq, Nk, heads, hd};
        if (tc)
            mgv::attn_fwd_tc(p, static_cast<cudaStream_t>(stream));
        else
            mgv::attn_fwd_simt<__nv_bfloat16>(p, static_cast<cudaStream_t>(stream));
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}
int mgv_dev_attn_bwd(int tc, const void* q, int64_t q_ld, const void* k, int64_t k_ld, const void* v, int64_t v_ld,
                     const void* o, int64_t o_ld, const float* lse, const void* dO, int64_t do_ld, float* Dvec,
                     void* dq, int64_t dq_ld, void* dk, int64_t dk_ld, void* dv, int64_t dv_ld, float* dkv_part,
                     int q_splits, int Nq, int Nk, int heads, int hd, void* stream) {
    try {
        mgv::AttnBwdProblem p{mgv::AttnProblem{q, q_ld, k, k_ld, v, v_ld, const_cast<void*>(o), o_ld,
                                               const_cast<float*>(lse), Nq, Nk, heads, hd},
                              dO, do_ld, Dvec, dq, dq_ld, dk, dk_ld, dv, dv_ld, dkv_part, q_splits};
        if (tc)
            mgv::attn_bwd_tc(p, static_cast<cudaStream_t>(stream));
        else
            mgv::attn_bwd_simt<__nv_bfloat16>(p, static_cast<cudaStream_t>(stream));
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}
}
