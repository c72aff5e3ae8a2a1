// tcgen05 flash attention for sm_100a (bf16 operands, fp32 softmax/accumulate).
//
// Forward, one CTA per (128-query tile, head):
//   warp 0      TMA producer: Q once, then K/V tiles through a 2-stage ring
//   warp 1      MMA issuer:   S_j = Q K_j^T into one of two TMEM S buffers,
//                             O += P_{j-1} V_{j-1} into the TMEM O accumulator
//   warp 2      TMEM allocator (512 columns: S0 | S1 | O)
//   warps 4..7  softmax, one thread per query row (thread i <-> TMEM lane i):
//               tcgen05.ld S -> online softmax in the log2 domain (ex2.approx)
//               -> P (bf16) to shared memory -> signal the PV MMA.  O is
//               rescaled in TMEM only when the running max grows by > 2^8
//               (stale-max trick), then normalised in the epilogue.
//
// head_dim is not a power of two in the 10B shape (144 = 64 + 64 + 16): Q/K/V
// tiles are stored as 64-column chunks with the 128-byte swizzle plus a
// 16-column tail with the 32-byte swizzle; S = Q K^T walks K-steps across the
// chunks, and O = P V is issued as an N=128 MMA (V read as an MN-major operand
// from the same smem tile) plus an N=16 MMA for the tail.  No transposed
// copies of K or V are ever made.
#include <cfloat>

#include "attn.h"
#include "gemm.cuh"
#include "ptx.cuh"

namespace mgv {

namespace {

constexpr int BM = 128;  // queries per CTA
constexpr int BN = 128;  // keys per tile
constexpr float kLog2e = 1.4426950408889634f;

template <int HD>
struct AttnCfg {
    static constexpr int NF = HD / 64;           // full 64-column chunks
    static constexpr int TAIL = HD % 64;         // 0 or 16
    static_assert(TAIL == 0 || TAIL == 16, "head_dim must be 64k or 64k+16");
    static constexpr int TILE = NF * 16384 + (TAIL ? 4096 : 0);  // bytes of a 128 x HD bf16 tile
    static constexpr int P_BYTES = 2 * 16384;                     // 128 x 128 bf16, two SW128 chunks
    static constexpr int SMEM = TILE /*Q*/ + 2 * TILE /*K*/ + 2 * TILE /*V*/ + P_BYTES + 1024 + 256;
    static constexpr int O_COL = 256;  // TMEM column of the O accumulator
};

struct TmapSet {
    CUtensorMap q128, q32, k128, k32, v128, v32;
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int HD>
__device__ __forceinline__ void load_tile(uint8_t* dst, const CUtensorMap* m128, const CUtensorMap* m32,
                                          uint64_t* bar, int col0, int row0) {
    using C = AttnCfg<HD>;
#pragma unroll
    for (int c = 0; c < C::NF; ++c) tma_load_2d(dst + c * 16384, m128, bar, col0 + c * 64, row0);
    if (C::TAIL) tma_load_2d(dst + C::NF * 16384, m32, bar, col0 + C::NF * 64, row0);
}

}  // namespace

template <int HD>
__global__ void __launch_bounds__(256, 1) attn_fwd_tc_kernel(const __grid_constant__ TmapSet tm, AttnProblem p) {
    using C = AttnCfg<HD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + C::TILE;
    uint8_t* sV = sK + 2 * C::TILE;
    uint8_t* sP = sV + 2 * C::TILE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sP + C::P_BYTES);
    uint64_t* q_full = bars;
    uint64_t* k_full = bars + 1;    // [2]
    uint64_t* v_full = bars + 3;    // [2]
    uint64_t* kv_empty = bars + 5;  // [2]
    uint64_t* s_full = bars + 7;    // [2]
    uint64_t* s_empty = bars + 9;   // [2]
    uint64_t* p_full = bars + 11;
    uint64_t* pv_done = bars + 12;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int h = blockIdx.y, q0 = blockIdx.x * BM;
    const int nkv = (p.Nk + BN - 1) / BN;
    const int qcol = h * HD, kcol = h * HD, vcol = h * HD;

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&kv_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&s_empty[i], 4);
        }
        mbar_init(p_full, 4);
        mbar_init(pv_done, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (elect_one()) {
            tma_prefetch(&tm.q128);
            tma_prefetch(&tm.k128);
            tma_prefetch(&tm.v128);
            mbar_arrive_expect_tx(q_full, C::TILE);
            load_tile<HD>(sQ, &tm.q128, &tm.q32, q_full, qcol, q0);
            for (int j = 0; j < nkv; ++j) {
                const int st = j & 1;
                if (j >= 2) mbar_wait(&kv_empty[st], ((j - 2) >> 1) & 1);
                mbar_arrive_expect_tx(&k_full[st], C::TILE);
                load_tile<HD>(sK + st * C::TILE, &tm.k128, &tm.k32, &k_full[st], kcol, j * BN);
                mbar_arrive_expect_tx(&v_full[st], C::TILE);
                load_tile<HD>(sV + st * C::TILE, &tm.v128, &tm.v32, &v_full[st], vcol, j * BN);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        constexpr uint32_t idS = idesc_bf16_f32(BM, BN, false, false);
        constexpr uint32_t idO = idesc_bf16_f32(BM, C::NF >= 2 ? 128 : 64, false, true);
        constexpr uint32_t idT = idesc_bf16_f32(BM, 16, false, true);
        const uint32_t aQ = smem_u32(sQ), aP = smem_u32(sP);
        auto issue_S = [&](int j) {
            const int st = j & 1, sb = j & 1;
            const uint32_t aK = smem_u32(sK + st * C::TILE);
            const uint32_t d = tmem + sb * BN;
            int kk = 0;
#pragma unroll
            for (int c = 0; c < C::NF; ++c)
#pragma unroll
                for (int k = 0; k < 4; ++k, ++kk)
                    umma_f16_ss(d, smem_desc(aQ + c * 16384 + k * 32, 16, 1024, kSwizzle128),
                                smem_desc(aK + c * 16384 + k * 32, 16, 1024, kSwizzle128), idS, kk > 0);
            if (C::TAIL)
                umma_f16_ss(d, smem_desc(aQ + C::NF * 16384, 16, 256, kSwizzle32),
                            smem_desc(aK + C::NF * 16384, 16, 256, kSwizzle32), idS, 1);
        };
        auto issue_PV = [&](int j) {
            const int st = j & 1;
            const uint32_t aV = smem_u32(sV + st * C::TILE);
            const uint32_t d = tmem + C::O_COL;
#pragma unroll
            for (int ks = 0; ks < BN / 16; ++ks) {
                // A = P (K-major over kv): chunk ks/4, 32-byte step inside the 128B atom
                const uint64_t ad = smem_desc(aP + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024, kSwizzle128);
                const uint32_t acc = (j > 0 || ks > 0) ? 1u : 0u;
                if (C::NF >= 2) {
                    // columns 0..127 of O: V chunks 0,1 as an MN-major operand (LBO = chunk stride)
                    umma_f16_ss(d, ad, smem_desc(aV + ks * 2048, 16384, 1024, kSwizzle128), idO, acc);
                    if (C::NF >= 3)  // not used for HD <= 191
                        umma_f16_ss(d + 128, ad, smem_desc(aV + 2 * 16384 + ks * 2048, 16384, 1024, kSwizzle128),
                                    idesc_bf16_f32(BM, 64, false, true), acc);
                } else {
                    umma_f16_ss(d, ad, smem_desc(aV + ks * 2048, 16384, 1024, kSwizzle128), idO, acc);
                }
                if (C::TAIL)
                    umma_f16_ss(d + C::NF * 64, ad, smem_desc(aV + C::NF * 16384 + ks * 512, 0, 256, kSwizzle32), idT,
                                acc);
            }
        };
        mbar_wait(q_full, 0);
        for (int j = 0; j < nkv; ++j) {
            const int st = j & 1;
            mbar_wait(&k_full[st], (j >> 1) & 1);
            if (j >= 2) mbar_wait(&s_empty[st], ((j - 2) >> 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                issue_S(j);
                umma_commit(&s_full[st]);
            }
            __syncwarp();
            if (j >= 1) {
                mbar_wait(p_full, (j - 1) & 1);
                mbar_wait(&v_full[(j - 1) & 1], ((j - 1) >> 1) & 1);
                tc_fence_after();
                if (elect_one()) {
                    issue_PV(j - 1);
                    umma_commit(pv_done);
                    umma_commit(&kv_empty[(j - 1) & 1]);
                }
                __syncwarp();
            }
        }
        if (nkv > 0) {
            const int j = nkv - 1;
            mbar_wait(p_full, j & 1);
            mbar_wait(&v_full[j & 1], (j >> 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                issue_PV(j);
                umma_commit(pv_done);
                umma_commit(&kv_empty[j & 1]);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ softmax (thread = query row)
        const int wq = warp - 4;
        const int row = wq * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
        float m2 = -FLT_MAX;  // running max, log2 domain
        float l = 0.0f;
        for (int j = 0; j < nkv; ++j) {
            const int sb = j & 1;
            mbar_wait(&s_full[sb], (j >> 1) & 1);
            tc_fence_after();
            float s[BN];
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) tmem_ld32(tmem + lane_base + sb * BN + c * 32, reinterpret_cast<uint32_t*>(s + c * 32));
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_empty[sb]);
            const int kv0 = j * BN;
            float mx = -FLT_MAX;
#pragma unroll
            for (int c = 0; c < BN; ++c) {
                s[c] = (kv0 + c < p.Nk) ? s[c] * kLog2e : -FLT_MAX;
                mx = fmaxf(mx, s[c]);
            }
            float alpha = 1.0f, m_use = m2;
            if (j == 0) {
                m_use = mx;
            } else if (mx > m2 + 8.0f) {
                m_use = mx;
                alpha = ex2(m2 - mx);
            }
            float ps = 0.0f;
            uint32_t pk[BN / 2];
#pragma unroll
            for (int c = 0; c < BN; c += 2) {
                const float p0 = ex2(s[c] - m_use), p1 = ex2(s[c + 1] - m_use);
                ps += p0 + p1;
                pk[c / 2] = pack_bf16(p0, p1);
            }
            if (j >= 1) {
                mbar_wait(pv_done, (j - 1) & 1);  // PV_{j-1} done: O stable, P buffer free
                tc_fence_after();
                if (__any_sync(0xffffffff, alpha != 1.0f)) {
                    const uint32_t ob = tmem + lane_base + C::O_COL;
#pragma unroll 1
                    for (int c = 0; c < HD / 16; ++c) {
                        uint32_t r[16];
                        tmem_ld16(ob + c * 16, r);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 16; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
                        tmem_st16(ob + c * 16, r);
                    }
                    tmem_wait_st();
                }
            }
            l = l * alpha + ps;
            m2 = m_use;
            // P row -> smem, SW128 K-major: 16-byte unit u of row r lives at (u ^ (r & 7))
#pragma unroll
            for (int u = 0; u < BN / 8; ++u) {
                const int chunk = u >> 3, uu = u & 7;
                uint8_t* dst = sP + chunk * 16384 + row * 128 + ((uu ^ (row & 7)) << 4);
                *reinterpret_cast<uint4*>(dst) = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
            }
            fence_proxy_async();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(p_full);
        }
        // epilogue: O / l -> global (token-major), lse
        if (nkv > 0) {
            mbar_wait(pv_done, (nkv - 1) & 1);
            tc_fence_after();
        }
        const int q = q0 + row;
        const float inv = l > 0.0f ? 1.0f / l : 0.0f;
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.o) + (int64_t)q * p.o_ld + h * HD;
#pragma unroll 1
        for (int c = 0; c < HD / 16; ++c) {
            uint32_t r[16];
            tmem_ld16(tmem + lane_base + C::O_COL + c * 16, r);
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
        if (q < p.Nq) p.lse[(int64_t)h * p.Nq + q] = (m2 + __log2f(l)) * 0.6931471805599453f;
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
static void launch_fwd(const AttnProblem& p, cudaStream_t s) {
    using C = AttnCfg<HD>;
    TmapSet tm;
    // operands are token-major (rows = tokens, ld = row stride in elements)
    const uint64_t qc = (uint64_t)p.heads * HD, kc = qc, vc = qc;
    make_tmap_sw(&tm.q128, p.q, qc, p.Nq, p.q_ld, 64, BM, CU_TENSOR_MAP_SWIZZLE_128B);
    make_tmap_sw(&tm.q32, p.q, qc, p.Nq, p.q_ld, 16, BM, CU_TENSOR_MAP_SWIZZLE_32B);
    make_tmap_sw(&tm.k128, p.k, kc, p.Nk, p.k_ld, 64, BN, CU_TENSOR_MAP_SWIZZLE_128B);
    make_tmap_sw(&tm.k32, p.k, kc, p.Nk, p.k_ld, 16, BN, CU_TENSOR_MAP_SWIZZLE_32B);
    make_tmap_sw(&tm.v128, p.v, vc, p.Nk, p.v_ld, 64, BN, CU_TENSOR_MAP_SWIZZLE_128B);
    make_tmap_sw(&tm.v32, p.v, vc, p.Nk, p.v_ld, 16, BN, CU_TENSOR_MAP_SWIZZLE_32B);
    static bool set = false;
    if (!set) {
        MGV_CUDA(cudaFuncSetAttribute(attn_fwd_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
        set = true;
    }
    dim3 grid((p.Nq + BM - 1) / BM, p.heads);
    attn_fwd_tc_kernel<HD><<<grid, 256, C::SMEM, s>>>(tm, p); ::mgv::note_launch();
    MGV_CUDA(cudaGetLastError());
}

void attn_fwd_tc(const AttnProblem& p, cudaStream_t s) {
    switch (p.hd) {
        case 64: launch_fwd<64>(p, s); break;
        case 128: launch_fwd<128>(p, s); break;
        case 144: launch_fwd<144>(p, s); break;
        default: throw std::runtime_error("attn_fwd_tc: unsupported head_dim");
    }
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
